# Round-end evidence on the final build (one GPU): smoke, every GPU test, the bench
# lines, the reference arm, the ncu launch list of the default bench, one full capture of
# k_adam / k_pack in the default mode, and compute-sanitizer over the smoke path.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
bash tools/gpu_round.sh > gpurun_out/round.log 2>&1
tail -30 gpurun_out/round.log
B="python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k regex:'k_adam$|k_pack' -s 60 -c 3 -o gpurun_out/prof_adam $B > gpurun_out/ncu_adam.log 2>&1
tail -n 2 gpurun_out/ncu_adam.log
bash tools/sanitize.sh 2>&1 | tail -20
