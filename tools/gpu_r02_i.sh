set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --durations=5 2>&1 | tail -12 | tee gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; tail -1 gpurun_out/bench_$name.err; }
run 11m --config 11m --moments persist --no-cpu-baseline --no-e2e
run 11m_sync --config 11m --moments persist --no-cpu-baseline --no-e2e --sync-activate
run 100m_persist --config 100m --moments persist --no-cpu-baseline --warmup 100 --steps 100
run default --steps 20 --warmup 5
run default_sync --steps 20 --warmup 5 --sync-activate --no-persist-detail --no-cpu-baseline
run fine_refresh --fine-filter --refresh-bounds --no-cpu-baseline --steps 20 --warmup 5
