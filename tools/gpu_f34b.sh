# f3 (coalesced SSD I/O) + f4 (device-side Lloyd loop): parity and bench.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 900 python -m pytest tests/test_gpu_order.py tests/test_gpu_store.py -x -q --durations=5 2>&1 | tail -12 | tee gpurun_out/pytest_f34.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; python tools/jline.py gpurun_out/bench_$name.json; tail -2 gpurun_out/bench_$name.err; }
run tsp --config 300m_tsp --no-cpu-baseline
run store1b --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e
run store1b_t16 --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e --io-threads 16
run store1b_t4 --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e --io-threads 4
