# GPU tests touched this round (store format 2, multirank C1/C2), then a k_xfer
# CTA / buffer sweep on the default bench (driver window: warmup 5, steps 20).
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 1200 python -m pytest tests/test_gpu_store.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -x -q 2>&1 | tail -8 | tee gpurun_out/pytest_tune.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; tail -1 gpurun_out/bench_$name.err; }
for cfg in "8 4 4 4" "16 1 4 4" "16 2 4 2" "32 1 3 4" "12 2 6 3" "24 2 3 2" "8 2 6 6"; do
  set -- $cfg
  TGS_GATHER_CTAS=$1 TGS_SCATTER_CTAS=$2 TGS_GATHER_BUFS=$3 TGS_SCATTER_BUFS=$4 run t_g$1_s$2_b$3_$4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e
done
