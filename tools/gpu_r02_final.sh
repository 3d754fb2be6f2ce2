# Round-2 evidence on the final build (one GPU): smoke, every GPU test, the bench lines,
# the reference arm, the ncu launch list of the default bench, sanitizers over smoke.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -25 | tee gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; tail -1 gpurun_out/bench_$name.err; }
run default_w5 --steps 20 --warmup 5
run default_w5_b --steps 20 --warmup 5 --no-cpu-baseline --no-persist-detail
run default
run 11m --config 11m --moments persist --no-cpu-baseline
run 1b_shard8 --config 1b --shard-of 8 --warmup 30
run fine_refresh --fine-filter --refresh-bounds --no-cpu-baseline --no-persist-detail --steps 20 --warmup 5
run 300m_tsp --config 300m_tsp --no-cpu-baseline --no-persist-detail
run store_1b_shard8 --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; tail -c 400 gpurun_out/bench_reference.json
TGS_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config 100m --moments persist --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; python tools/jline.py gpurun_out/bench_gloo2.json
B="python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e --no-persist-detail"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches_bench.log 2>&1
echo "ncu launches rc=$?"
echo "compute-sanitizer: closed on this pool (not run)"
