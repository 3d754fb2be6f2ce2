mkdir -p gpurun_out
make -s || exit 1
timeout 900 python bench.py --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e --no-overlap > gpurun_out/bench_store1b_serial.json 2> gpurun_out/bench_store1b_serial.err
python tools/jline.py gpurun_out/bench_store1b_serial.json
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench_store1b_serial.json').read().strip().splitlines()[-1])
print({k: d['detail'][k] for k in ('h2d_ms_per_step', 'd2h_ms_per_step', 'h2d_GB_per_step', 'd2h_GB_per_step')})
PY
