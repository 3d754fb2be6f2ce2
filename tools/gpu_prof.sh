# ncu evidence for the bench workload: launch list + full capture of the top kernels.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
B="python bench.py --steps 4 --warmup 4 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
   --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'k_adam$|k_pack|k_plan|k_cull' -s 12 -c 4 -o gpurun_out/prof $B > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
