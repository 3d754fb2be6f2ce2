# A/B on one box: A lists released after Adam(t)'s prologue (default) vs after the whole Adam
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 600 env "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; python tools/jline.py gpurun_out/bench_$name.json; }
for i in 1 2; do
  run ab_early$i TGS_LISTS_AFTER_ADAM=0 python bench.py --no-cpu-baseline --no-e2e
  run ab_late$i TGS_LISTS_AFTER_ADAM=1 python bench.py --no-cpu-baseline --no-e2e
done
run ab_early_g8 TGS_LISTS_AFTER_ADAM=0 python bench.py --config 1b --shard-of 8 --no-cpu-baseline --no-e2e --warmup 30
run ab_late_g8 TGS_LISTS_AFTER_ADAM=1 python bench.py --config 1b --shard-of 8 --no-cpu-baseline --no-e2e --warmup 30
