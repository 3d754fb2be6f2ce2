# ncu evidence for the bench workload: launch list of the bench command + one
# full capture of each hot kernel; the f4 kernels on the shuffled 300m views;
# the SSD roofline of the f3 store's access pattern.  One GPU (never multi-rank).
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
B="python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches_bench.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on \
   -k regex:'k_adam$|k_adam_prologue|k_pack|k_plan|k_cull|k_quota|k_evict|k_readmit|k_fine|k_refresh' -s 170 -c 12 -o gpurun_out/prof $B --fine-filter --refresh-bounds > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'k_assign|k_update|k_inner_tour|k_cluster_tour|k_init_step|k_members|k_lex' -s 2 -c 10 -o gpurun_out/prof_order \
   python -c "
import sys; sys.path.insert(0, '.')
import workload as W
from paper_2605_20150_b200 import tidegs as T
wl = W.CONFIGS['300m_random']; sc = wl.scene(); tr = wl.trajectory(sc)
p = T.order_views(tr.features(150.0))
print('order', p[2], p[3], p[4], 'ms')
" > gpurun_out/ncu_order.log 2>&1
tail -3 gpurun_out/ncu_order.log
timeout 600 python tools/ssd_probe.py /tmp/ssd_probe.bin 966656 8 2>&1 | tee gpurun_out/ssd_probe.txt
rm -f /tmp/ssd_probe.bin
