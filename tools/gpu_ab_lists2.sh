# list release after Adam's prologue vs after Adam, in the chain-bound configs (11m, 100m persist)
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 600 env "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo -n "$name "; python tools/jline.py gpurun_out/bench_$name.json | cut -c1-90; }
for r in 1 2; do
run l2_late_11m$r TGS_LISTS_AFTER_ADAM=1 python bench.py --config 11m --moments persist --no-cpu-baseline --no-e2e --steps 200
run l2_early_11m$r TGS_LISTS_AFTER_ADAM=0 python bench.py --config 11m --moments persist --no-cpu-baseline --no-e2e --steps 200
run l2_late_100m$r TGS_LISTS_AFTER_ADAM=1 python bench.py --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 400 --steps 100
run l2_early_100m$r TGS_LISTS_AFTER_ADAM=0 python bench.py --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 400 --steps 100
done
