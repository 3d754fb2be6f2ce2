# five write-back ring slots on the flat tier: full GPU suite, then A/B vs three (previous build)
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2700 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/rings_$name.json 2> gpurun_out/rings_$name.err; echo "$name $(python tools/jline.py gpurun_out/rings_$name.json)"; }
P=$PWD/paper_2605_20150_b200/libtidegs_prev.so
for r in 1 2; do
run new_w5_$r --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
TGS_LIB=$P run prev_w5_$r --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
done
run new_w20 --no-cpu-baseline --no-persist-detail --no-e2e
TGS_LIB=$P run prev_w20 --no-cpu-baseline --no-persist-detail --no-e2e
run new_100m --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
TGS_LIB=$P run prev_100m --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
run new_1b --config 1b --shard-of 8 --no-cpu-baseline --no-e2e --warmup 30
TGS_LIB=$P run prev_1b --config 1b --shard-of 8 --no-cpu-baseline --no-e2e --warmup 30
