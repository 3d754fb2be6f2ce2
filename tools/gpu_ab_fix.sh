# fix-up stream (k_readmit) at the highest priority vs the default, same box
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 600 env "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo -n "$name "; python tools/jline.py gpurun_out/bench_$name.json; }
for r in 1 2; do
run fx_hi_100m$r TGS_FIX_PRIO=1 python bench.py --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 400 --steps 100
run fx_lo_100m$r TGS_FIX_PRIO=0 python bench.py --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 400 --steps 100
done
run fx_hi_def TGS_FIX_PRIO=1 python bench.py --no-cpu-baseline --no-e2e
run fx_lo_def TGS_FIX_PRIO=0 python bench.py --no-cpu-baseline --no-e2e
