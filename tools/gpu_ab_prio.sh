# A/B on one box: plan stream at the highest priority (default) vs the default priority
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 600 env "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo -n "$name "; python tools/jline.py gpurun_out/bench_$name.json; }
for i in 1 2; do
  run pr_hi$i TGS_PLAN_PRIO=1 python bench.py --no-cpu-baseline --no-e2e
  run pr_lo$i TGS_PLAN_PRIO=0 python bench.py --no-cpu-baseline --no-e2e
done
run pr_hi_100m TGS_PLAN_PRIO=1 python bench.py --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 400 --steps 100
run pr_lo_100m TGS_PLAN_PRIO=0 python bench.py --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 400 --steps 100
run pr_hi_inf TGS_PLAN_PRIO=1 python bench.py --config 1b --shard-of 8 --capacity 244141 --pool-slots 30518 --no-cpu-baseline --no-e2e --warmup 100
run pr_lo_inf TGS_PLAN_PRIO=0 python bench.py --config 1b --shard-of 8 --capacity 244141 --pool-slots 30518 --no-cpu-baseline --no-e2e --warmup 100
