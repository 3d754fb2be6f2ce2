# 3 write-back ring slots, small plan CTAs, f1/f2 folded into k_adam: GPU tests,
# then the default bench, a transfer-CTA sweep, and the chain-bound / f1-f2 configs.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -16 | tee gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; tail -1 gpurun_out/bench_$name.err; }
run default --steps 20 --warmup 5 --no-persist-detail
for cfg in "8 2 6 6" "12 2 4 4" "16 2 4 4" "8 1 6 6" "16 1 6 6"; do
  set -- $cfg
  TGS_GATHER_CTAS=$1 TGS_SCATTER_CTAS=$2 TGS_GATHER_BUFS=$3 TGS_SCATTER_BUFS=$4 run t_g$1_s$2_b$3_$4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e
done
run 11m --config 11m --moments persist --no-cpu-baseline --no-e2e
run 100m_persist --config 100m --moments persist --no-cpu-baseline --warmup 100 --steps 100
run fine_refresh --fine-filter --refresh-bounds --no-cpu-baseline --steps 20 --warmup 5
