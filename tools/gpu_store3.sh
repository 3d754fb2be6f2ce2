set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 900 python -m pytest tests/test_gpu_store.py -x -q --durations=4 2>&1 | tail -8 | tee gpurun_out/pytest_store3.log
