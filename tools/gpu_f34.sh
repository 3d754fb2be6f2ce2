# f3 tuning sweep + f4 parity and bench on one GPU.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 900 python -m pytest tests/test_gpu_order.py -x -q --durations=5 2>&1 | tail -12 | tee gpurun_out/pytest_order.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; python tools/jline.py gpurun_out/bench_$name.json; tail -2 gpurun_out/bench_$name.err; }
run tsp --config 300m_tsp --no-cpu-baseline
run store1b_t8 --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e --io-threads 8
run store1b_t32 --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e --io-threads 32
run store1b_h8c --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e --io-threads 32 --cache-blocks 21032
