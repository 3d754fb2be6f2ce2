set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_store.py -x -q 2>&1 | tail -3
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; python tools/jline.py gpurun_out/bench_$name.json; }
run a3_default --no-cpu-baseline
run a3_g8 --config 300m --shard-of 8 --no-cpu-baseline --no-e2e
run a3_g4 --config 300m --shard-of 4 --no-cpu-baseline --no-e2e
run a3_1b --config 1b --shard-of 8 --no-cpu-baseline --warmup 30
