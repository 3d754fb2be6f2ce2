set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 600 python -m pytest tests/test_gpu_order.py -x -q -k "not 100m" 2>&1 | tail -2
python - <<'PY'
import sys; sys.path.insert(0, '.')
import workload as W
from paper_2605_20150_b200 import tidegs as T
wl = W.CONFIGS['300m_random']; sc = wl.scene(); tr = wl.trajectory(sc)
f = tr.features(150.0)
for i in range(3):
    p = T.order_views(f)
    print('order k', p[2], 'lloyd', p[3], 'gpu_ms', round(p[4], 2))
PY
TGS_TRACE=1 timeout 600 python bench.py --config 300m --shard-of 8 --steps 8 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/trace8.json 2> gpurun_out/trace8.err
python tools/jline.py gpurun_out/trace8.json
grep "tgs trace" gpurun_out/trace8.err | tail -60
