set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
TGS_TRACE=1 timeout 900 python bench.py --steps 6 --warmup 45 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/trace_bench.json 2> gpurun_out/trace.txt
tail -c 1500 gpurun_out/trace_bench.json
