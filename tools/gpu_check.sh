# One GPU call: build, smoke, gpu tests, bench.  Outputs land in gpurun_out/.
set -o pipefail
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20 | tee gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q --durations=15 ${PYTEST_ARGS} 2>&1 | tail -40 | tee gpurun_out/pytest_gpu.log
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py $BENCH 2>&1 | tail -5 | tee gpurun_out/bench.log
fi
