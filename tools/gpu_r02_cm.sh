# k_commit on its own stream, double-buffered stage_in: CE parity, then A/B vs the previous build
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "xfer or _ce or 300m or 1b or writeback or readmission" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err; echo "$name $(python tools/jline.py gpurun_out/ab_$name.json)"; }
for r in 1 2 3; do
run new_w5_$r --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
TGS_LIB=$PWD/paper_2605_20150_b200/libtidegs_prev.so run prev_w5_$r --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
done
run new_w20 --no-cpu-baseline --no-persist-detail --no-e2e
TGS_LIB=$PWD/paper_2605_20150_b200/libtidegs_prev.so run prev_w20 --no-cpu-baseline --no-persist-detail --no-e2e
run new_100m --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
TGS_LIB=$PWD/paper_2605_20150_b200/libtidegs_prev.so run prev_100m --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
