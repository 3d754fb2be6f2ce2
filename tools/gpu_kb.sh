set -o pipefail
mkdir -p gpurun_out
for v in "" _m2 _m4; do
  echo "== variant libtidegs$v.so"
  TGS_LIB=$PWD/paper_2605_20150_b200/libtidegs$v.so timeout 300 python tools/kbench.py 3000 20 2>&1 | tail -2
done | tee gpurun_out/kbench.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "tiny or masked or nonfinite" 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
