# same-box A/B of the a4 transfer mechanism (copy-engine runs vs TMA kernels), alternating
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err; echo "$name $(python tools/jline.py gpurun_out/ab_$name.json)"; }
for r in 1 2 3; do
run ce_w5_$r --xfer ce --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
run kernel_w5_$r --xfer kernel --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
done
for r in 1 2; do
run ce_w20_$r --xfer ce --no-cpu-baseline --no-persist-detail --no-e2e
run kernel_w20_$r --xfer kernel --no-cpu-baseline --no-persist-detail --no-e2e
done
run ce_1b --xfer ce --config 1b --shard-of 8 --no-cpu-baseline --no-e2e --warmup 30
run kernel_1b --xfer kernel --config 1b --shard-of 8 --no-cpu-baseline --no-e2e --warmup 30
run ce_100m --xfer ce --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
run kernel_100m --xfer kernel --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
