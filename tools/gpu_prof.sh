# ncu evidence for the bench workload: launch list of the bench command + one
# full capture of each hot kernel.  Run on one GPU (never multi-rank).
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "writeback or readmission" 2>&1 | tail -3 | tee gpurun_out/pytest_new.log
B="python bench.py --steps 6 --warmup 30 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k regex:'k_adam$|k_pack|k_plan|k_cull|k_evict|k_cold_init|k_quota' -s 200 -c 8 -o gpurun_out/prof $B > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
