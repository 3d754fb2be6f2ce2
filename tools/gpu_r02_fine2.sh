# k_fine: first camera's planes in registers (new) vs per-row smem planes (prev), same launches
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "fine or level2" 2>&1 | tail -1
B="python bench.py --fine-filter --refresh-bounds --steps 4 --warmup 30 --no-cpu-baseline --no-e2e --no-persist-detail"
for v in new prev; do
  if [ $v = prev ]; then export TGS_LIB=$PWD/paper_2605_20150_b200/libtidegs_prev.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,dram__bytes_read.sum -k regex:'k_fine' -s 25 -c 3 $B 2>&1 | grep -E "gpu__time|l1tex|dram" | sed "s/^/$v /"
done
