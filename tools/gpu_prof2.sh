# default-mode k_adam capture (traffic), f4 kernels after the reduction fix,
# SSD probe with pinned vs pageable buffers on a 30 GiB file.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 600 python -m pytest tests/test_gpu_order.py -x -q -k "not 100m" 2>&1 | tail -3
B="python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k regex:'k_adam$|k_pack' -s 60 -c 3 -o gpurun_out/prof_adam $B > gpurun_out/ncu_adam.log 2>&1
tail -n 2 gpurun_out/ncu_adam.log
python - <<'PY' > gpurun_out/order_time.txt 2>&1
import sys; sys.path.insert(0, '.')
import workload as W
from paper_2605_20150_b200 import tidegs as T
wl = W.CONFIGS['300m_random']; sc = wl.scene(); tr = wl.trajectory(sc)
f = tr.features(150.0)
for i in range(3):
    p = T.order_views(f)
    print('order k', p[2], 'lloyd', p[3], 'gpu_ms', round(p[4], 2))
PY
cat gpurun_out/order_time.txt
timeout 900 ncu --set full --clock-control none -k regex:'k_assign|k_update|k_inner_tour|k_cluster_tour|k_init_step|k_members|k_lex|k_lloyd' -c 12 -o gpurun_out/prof_order2 \
   python -c "
import sys; sys.path.insert(0, '.')
import workload as W
from paper_2605_20150_b200 import tidegs as T
wl = W.CONFIGS['300m_random']; sc = wl.scene(); tr = wl.trajectory(sc)
T.order_views(tr.features(150.0))
" > gpurun_out/ncu_order2.log 2>&1
timeout 900 python tools/ssd_probe.py /tmp/ssd_probe.bin 966656 30 2>&1 | tee gpurun_out/ssd_probe2.txt
rm -f /tmp/ssd_probe.bin
