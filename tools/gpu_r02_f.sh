# all GPU tests; traces of the chain-bound configs; f1/f2; f3 with/without read-ahead;
# sanitizers on smoke; k_adam traffic capture with its step log
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 2700 python -m pytest tests -m gpu -q -x --durations=5 2>&1 | tail -10 | tee gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; tail -1 gpurun_out/bench_$name.err; }
TGS_TRACE=1 run trace_11m --config 11m --moments persist --no-cpu-baseline --no-e2e --warmup 20 --steps 20
grep "tgs trace" gpurun_out/bench_trace_11m.err | tail -80 > gpurun_out/trace_11m.txt
TGS_TRACE=1 run trace_100m --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 20
grep "tgs trace" gpurun_out/bench_trace_100m.err | tail -100 > gpurun_out/trace_100m.txt
run fine_refresh --fine-filter --refresh-bounds --no-cpu-baseline --steps 20 --warmup 5
run store_1b_pf0 --config 1b --shard-of 8 --store /tmp/tgs_store --prefetch 0 --no-cpu-baseline --no-e2e
run store_1b_pf --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e
bash tools/sanitize.sh > gpurun_out/sanitize.log 2>&1; tail -12 gpurun_out/sanitize.log
B="python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e --no-persist-detail"
TGS_BENCH_STEPLOG=gpurun_out/steplog_r02.jsonl timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_adam<' -s 25 -c 1 -o gpurun_out/prof_adam_r02 $B > gpurun_out/ncu_adam.log 2>&1
tail -2 gpurun_out/ncu_adam.log
ncu -i gpurun_out/prof_adam_r02.ncu-rep --page raw --csv > gpurun_out/ncu_adam_raw_r02.csv 2>/dev/null; ls -la gpurun_out/ncu_adam_raw_r02.csv
