# ncu evidence for the bench workload: launch list of the bench command + one
# full capture of each hot kernel.  Run on one GPU (never multi-rank).
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
B="python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches_bench.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on \
   -k regex:'k_adam$|k_pack|k_plan|k_cull|k_fine|k_refresh' -s 170 -c 6 -o gpurun_out/prof $B --fine-filter --refresh-bounds > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
