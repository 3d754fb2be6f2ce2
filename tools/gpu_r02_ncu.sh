# ncu evidence on HEAD (copy-engine transfers): launch list of the default bench, one full
# capture of k_adam (step 30, with the step log giving its algorithmic bytes) and k_commit,
# one of k_fine / k_refresh in the --fine-filter --refresh-bounds run.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
B="python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e --no-persist-detail"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches_bench.log 2>&1
echo "launches rc=$?"
TGS_BENCH_STEPLOG=gpurun_out/steplog_cold.jsonl timeout 1500 ncu --set full --clock-control none --import-source on \
   -k regex:'k_adam$|k_commit' -s 58 -c 4 -o gpurun_out/prof_adam_commit python bench.py --steps 4 --warmup 30 --no-cpu-baseline --no-e2e --no-persist-detail > gpurun_out/ncu_adam.log 2>&1
tail -n 2 gpurun_out/ncu_adam.log
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k regex:'k_fine|k_refresh' -s 50 -c 2 -o gpurun_out/prof_fine python bench.py --fine-filter --refresh-bounds --steps 4 --warmup 30 --no-cpu-baseline --no-e2e --no-persist-detail > gpurun_out/ncu_fine.log 2>&1
tail -n 2 gpurun_out/ncu_fine.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; }
run fine_refresh --fine-filter --refresh-bounds --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
run fine --fine-filter --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
run 11m --config 11m --moments persist --no-cpu-baseline --no-e2e
