set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 900 python -m pytest tests/test_gpu_store.py -x -q 2>&1 | tail -3 | tee gpurun_out/pytest_store2.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; python tools/jline.py gpurun_out/bench_$name.json; tail -2 gpurun_out/bench_$name.err; }
run store1b_c --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline
run store1b_c4 --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e --io-threads 4
run store100m_c --config 100m --store /tmp/tgs_store --no-cpu-baseline --no-e2e
