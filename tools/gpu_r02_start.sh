# Round-2 opening evidence on HEAD: smoke, GPU tests, default bench, ncu launch list.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/linkbench tools/linkbench.cu && timeout 300 tools/linkbench > gpurun_out/linkbench.txt 2>&1; cat gpurun_out/linkbench.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -25 | tee gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python tools/jline.py gpurun_out/bench_default.json
