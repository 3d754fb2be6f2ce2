# f3 evidence on one GPU: store-tier parity tests, the full GPU suite, and
# bench lines with the shard on local disk below a CPU cache.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 1200 python -m pytest tests/test_gpu_store.py -x -q --durations=8 2>&1 | tail -30 | tee gpurun_out/pytest_store.log
if [ -n "$FULL" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 | tee gpurun_out/pytest_gpu.log
fi
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; tail -c 1500 gpurun_out/bench_$name.json; echo; tail -3 gpurun_out/bench_$name.err; }
if [ -n "$BENCH" ]; then
  run store_100m --config 100m --store /tmp/tgs_store --no-cpu-baseline --no-e2e
  run store_1b_shard8 --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e
fi
df -h /tmp | tail -1
