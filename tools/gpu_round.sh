# Round evidence on one GPU: smoke, every GPU test, the default bench and the other configs.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -25 | tee gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; python tools/jline.py gpurun_out/bench_$name.json; tail -2 gpurun_out/bench_$name.err; }
run default
run fine --fine-filter --no-cpu-baseline
run 100m_persist --config 100m --moments persist --no-cpu-baseline --warmup 400 --steps 100
run 11m --config 11m --moments persist --no-cpu-baseline --no-e2e
run 300m_random --config 300m_random --no-cpu-baseline --no-e2e --steps 10 --warmup 5
run 300m_tsp --config 300m_tsp --no-cpu-baseline
run 1b_shard8 --config 1b --shard-of 8 --no-cpu-baseline --warmup 30
run store_1b_shard8 --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; tail -c 300 gpurun_out/bench_reference.json
