set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 2700 python -m pytest tests -m gpu -q --durations=5 2>&1 | tail -10 | tee gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; tail -1 gpurun_out/bench_$name.err; }
run default --steps 20 --warmup 5
run fine_refresh --fine-filter --refresh-bounds --no-cpu-baseline --steps 20 --warmup 5
run store_1b_pf --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e
run 11m --config 11m --moments persist --no-cpu-baseline --no-e2e
B="python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e --no-persist-detail"
TGS_BENCH_STEPLOG=gpurun_out/steplog_r02.jsonl timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'^k_adam' -s 50 -c 2 -o gpurun_out/prof_adam_r02 $B > gpurun_out/ncu_adam.log 2>&1
tail -2 gpurun_out/ncu_adam.log
ncu -i gpurun_out/prof_adam_r02.ncu-rep --page raw --csv > gpurun_out/ncu_adam_raw_r02.csv 2>/dev/null; ls -la gpurun_out/ncu_adam_raw_r02.csv
