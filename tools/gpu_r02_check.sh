# HEAD check on one GPU: smoke, every GPU test, the default bench line.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --durations=15 2>&1 | tail -40 | tee gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; python tools/jline.py gpurun_out/bench_default.json; tail -2 gpurun_out/bench_default.err
