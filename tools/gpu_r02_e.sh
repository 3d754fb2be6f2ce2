# geo6 f1/f2 path: GPU tests, then the benches incl. early list release A/B
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=6 2>&1 | tail -12 | tee gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; tail -1 gpurun_out/bench_$name.err; }
run fine_refresh --fine-filter --refresh-bounds --no-cpu-baseline --steps 20 --warmup 5
run default_lists_late --steps 20 --warmup 5 --no-persist-detail --no-cpu-baseline
TGS_LISTS_AFTER_ADAM=0 run default_lists_early --steps 20 --warmup 5 --no-persist-detail --no-cpu-baseline
run 11m --config 11m --moments persist --no-cpu-baseline --no-e2e
TGS_LISTS_AFTER_ADAM=0 run 11m_early --config 11m --moments persist --no-cpu-baseline --no-e2e
run 100m_persist --config 100m --moments persist --no-cpu-baseline --warmup 100 --steps 100
TGS_LISTS_AFTER_ADAM=0 run 100m_persist_early --config 100m --moments persist --no-cpu-baseline --warmup 100 --steps 100
