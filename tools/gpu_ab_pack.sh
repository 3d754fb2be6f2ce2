# k_pack at 40 registers / 6 CTAs per SM (was 106 / 2) vs the previous build, same box
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "writeback or pipelined or tiny" 2>&1 | tail -2
L=$PWD/paper_2605_20150_b200
run() { name=$1; shift; timeout 600 env "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo -n "$name "; python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); det=d['detail']
print(round(d['value']/1e9,4), round(d['ms_per_step'],3), 'pack ms/step', round(det['evict_pack_ms_per_step'],4), 'S-dirty/step', det['churn']['evict_dirty_per_step'], 'adam', round(d['roofline']['frac'],3))" gpurun_out/bench_$name.json; }
for r in 1 2; do
run pk_new$r TGS_LIB=$L/libtidegs.so python bench.py --no-cpu-baseline --no-e2e
run pk_old$r TGS_LIB=$L/libtidegs_old.so python bench.py --no-cpu-baseline --no-e2e
done
run pk_new_rand TGS_LIB=$L/libtidegs.so python bench.py --config 300m_random --no-cpu-baseline --no-e2e --steps 10 --warmup 5
run pk_old_rand TGS_LIB=$L/libtidegs_old.so python bench.py --config 300m_random --no-cpu-baseline --no-e2e --steps 10 --warmup 5
timeout 900 ncu --set full --clock-control none -k regex:'k_pack' -s 10 -c 1 -o gpurun_out/prof_pack python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e > gpurun_out/ncu_pack.log 2>&1
tail -1 gpurun_out/ncu_pack.log
rm -f $L/libtidegs_old.so
