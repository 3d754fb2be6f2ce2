# k_adam without local-memory spills (R20 slow path out of line, step sizes in smem)
# vs the previous build (libtidegs_old.so), same box: kernel bench + step benches
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for r in 1 2; do
for v in "" _old; do
  echo -n "kbench libtidegs$v.so: "
  TGS_LIB=$PWD/paper_2605_20150_b200/libtidegs$v.so timeout 300 python tools/kbench.py 3000 20 2>&1 | grep k_adam
done
done
run() { name=$1; shift; timeout 600 env "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo -n "$name "; python tools/jline.py gpurun_out/bench_$name.json; }
L=$PWD/paper_2605_20150_b200
for r in 1 2; do
run ad_new$r TGS_LIB=$L/libtidegs.so python bench.py --no-cpu-baseline --no-e2e
run ad_old$r TGS_LIB=$L/libtidegs_old.so python bench.py --no-cpu-baseline --no-e2e
done
run ad_new_inf TGS_LIB=$L/libtidegs.so python bench.py --config 1b --shard-of 8 --capacity 244141 --pool-slots 30518 --no-cpu-baseline --no-e2e --warmup 100
run ad_old_inf TGS_LIB=$L/libtidegs_old.so python bench.py --config 1b --shard-of 8 --capacity 244141 --pool-slots 30518 --no-cpu-baseline --no-e2e --warmup 100
run ad_new_100m TGS_LIB=$L/libtidegs.so python bench.py --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 400 --steps 100
run ad_old_100m TGS_LIB=$L/libtidegs_old.so python bench.py --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 400 --steps 100
