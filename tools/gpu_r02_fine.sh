# k_fine (4 rows per thread, planes once per 4 rows): parity, timing; 11m dyn-qpw A/B
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -k "fine or pipelined or level2 or refresh" 2>&1 | tail -2
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json) fine_ms=$(python -c "import json;print(json.loads(open('gpurun_out/bench_$name.json').read().strip().splitlines()[-1])['detail']['fine_ms_per_step'])")"; }
run fine_refresh --fine-filter --refresh-bounds --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
for r in 1 2 3; do
TGS_ADAM_DYNQPW=1 run 11m_dyn_$r --config 11m --moments persist --no-cpu-baseline --no-e2e
TGS_ADAM_DYNQPW=0 run 11m_fix_$r --config 11m --moments persist --no-cpu-baseline --no-e2e
done
timeout 900 ncu --set full --clock-control none -k regex:'k_fine' -s 30 -c 1 -o gpurun_out/prof_fine2 python bench.py --fine-filter --refresh-bounds --steps 4 --warmup 30 --no-cpu-baseline --no-e2e --no-persist-detail > gpurun_out/ncu_fine2.log 2>&1; tail -1 gpurun_out/ncu_fine2.log
