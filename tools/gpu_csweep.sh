# SURVEY §8d capacity sweep: C = {1.25, 2.44, 5, max}x the mean #K_t estimate, cold restart.
# 300m on one GPU (the largest C that fits 180 GB with P = 36000 slots), and one GPU's share
# of the 8-way 1B table up to C_g = K_loc (the whole shard resident: no eviction ever).
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; python tools/jline.py gpurun_out/bench_$name.json; tail -1 gpurun_out/bench_$name.err; }
A="--no-cpu-baseline --no-e2e --warmup 100 --steps 50"
run cs_300m_1.25 --capacity 3233 $A
run cs_300m_2.44 $A
run cs_300m_5 --capacity 12930 $A
run cs_300m_10 --capacity 25860 --pool-slots 36000 $A
run cs_1b8_1.25 --config 1b --shard-of 8 --capacity 10776 $A
run cs_1b8_2.44 --config 1b --shard-of 8 $A
run cs_1b8_5 --config 1b --shard-of 8 --capacity 43080 $A
run cs_1b8_inf --config 1b --shard-of 8 --capacity 244141 --pool-slots 30518 $A
