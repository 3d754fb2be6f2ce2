# batched f1/f2 epilogue check, a timeline trace of the default bench, ncu evidence
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_store.py -q -x -k "fine or refresh or pipelined or store" 2>&1 | tail -4 | tee gpurun_out/pytest_c.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; }
TGS_TRACE=1 run trace --steps 8 --warmup 5 --no-cpu-baseline --no-e2e --no-persist-detail
grep "tgs trace" gpurun_out/bench_trace.err | tail -150 > gpurun_out/trace.txt
run fine_refresh --fine-filter --refresh-bounds --no-cpu-baseline --steps 20 --warmup 5
B="python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e --no-persist-detail"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
tail -2 gpurun_out/ncu_launches.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_adam|k_xfer' -s 120 -c 4 -o gpurun_out/prof_r02 $B > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
ncu -i gpurun_out/prof_r02.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw.csv 2>/dev/null; ls -la gpurun_out/ncu_full_raw.csv
