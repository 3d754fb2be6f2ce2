set -o pipefail
make -s || exit 1
for mp in -1 0.9 0.5 0.25; do echo "mask_p=$mp"; timeout 300 python tools/kbench.py 3000 20 $mp 2>&1 | tail -1; done | tee gpurun_out/kbench2.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "tiny or masked or nonfinite or fine" 2>&1 | tail -2
