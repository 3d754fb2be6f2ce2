# Round evidence on one GPU: tests, smoke, the default bench and the other configs.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -25 | tee gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; tail -c 600 gpurun_out/bench_$name.json; echo; }
run default
run fine --fine-filter --no-cpu-baseline
run 100m_persist --config 100m --moments persist --no-cpu-baseline --warmup 400 --steps 100
run 11m --config 11m --moments persist --no-cpu-baseline --no-e2e
run 300m_random --config 300m_random --no-cpu-baseline --no-e2e --steps 10 --warmup 5
