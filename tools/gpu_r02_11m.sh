# 11m chain-bound config: async parity tests, bench repeats, trace
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "pipelined or async or masked or fine" 2>&1 | tail -1; done
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; }
for r in 1 2 3; do run 11m_$r --config 11m --moments persist --no-cpu-baseline --no-e2e; done
TGS_TRACE=1 timeout 900 python bench.py --config 11m --moments persist --steps 12 --warmup 40 --no-cpu-baseline --no-e2e > gpurun_out/trace_11m.json 2> gpurun_out/trace_11m.txt
