# write-back kernels on their own stream: full GPU suite, then the chain-bound configs and the default
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
timeout 2700 python -m pytest tests -m gpu -q -x --durations=5 2>&1 | tail -12 | tee gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; }
for r in 1 2 3; do run 11m_$r --config 11m --moments persist --no-cpu-baseline --no-e2e; done
run 100m --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
run w5 --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
TGS_TRACE=1 timeout 900 python bench.py --config 11m --moments persist --steps 12 --warmup 40 --no-cpu-baseline --no-e2e > gpurun_out/trace_11m.json 2> gpurun_out/trace_11m.txt
