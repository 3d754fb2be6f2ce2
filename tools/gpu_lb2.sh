set -o pipefail
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/linkbench2 tools/linkbench2.cu || exit 1
timeout 300 tools/linkbench2 > gpurun_out/linkbench2.txt 2>&1; echo rc=$?
timeout 120 tools/linkbench2 tma > gpurun_out/linkbench2_tma.txt 2>&1; echo rc_tma=$?
cat gpurun_out/linkbench2.txt gpurun_out/linkbench2_tma.txt
