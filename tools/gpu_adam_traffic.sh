# k_adam traffic vs algorithmic bytes on the current build: one ncu --set full capture of
# the default (cold-restart) bench's k_adam at step 30, with the per-step fresh-row log
# that gives that launch's exact algorithmic bytes; and one in 100m persist (no fresh rows).
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_fresh.json 2> gpurun_out/bench_fresh.err
python tools/jline.py gpurun_out/bench_fresh.json
TGS_BENCH_STEPLOG=gpurun_out/steplog_cold.jsonl timeout 1500 ncu --set full --clock-control none --import-source on \
   -k regex:'k_adam$' -s 30 -c 1 -o gpurun_out/prof_adam_cold python bench.py --steps 4 --warmup 30 --no-cpu-baseline --no-e2e > gpurun_out/ncu_adam_cold.log 2>&1
tail -n 2 gpurun_out/ncu_adam_cold.log
TGS_BENCH_STEPLOG=gpurun_out/steplog_persist.jsonl timeout 1500 ncu --set full --clock-control none \
   -k regex:'k_adam$' -s 420 -c 1 -o gpurun_out/prof_adam_persist python bench.py --config 100m --moments persist --steps 4 --warmup 421 --no-cpu-baseline --no-e2e > gpurun_out/ncu_adam_persist.log 2>&1
tail -n 2 gpurun_out/ncu_adam_persist.log
