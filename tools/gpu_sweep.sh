# configs[4]: trajectory-locality sweep at 300M -- smooth vs random vs clustered-TSP order,
# one GPU's share of a G-way block-sharded table (G = 1, 2, 4, 8; --shard-of G)
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; python tools/jline.py gpurun_out/bench_$name.json; }
for G in 2 4 8; do
  run sweep_smooth_g$G --config 300m --shard-of $G --no-cpu-baseline --no-e2e
  run sweep_tsp_g$G --config 300m_tsp --shard-of $G --no-cpu-baseline --no-e2e
  run sweep_random_g$G --config 300m_random --shard-of $G --no-cpu-baseline --no-e2e --steps 10 --warmup 5
done
