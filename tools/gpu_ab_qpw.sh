# k_adam quads-per-warp adapted to small launches (>= 4 waves) vs fixed 16, same box
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
L=$PWD/paper_2605_20150_b200
run() { name=$1; shift; timeout 600 env "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo -n "$name "; python tools/jline.py gpurun_out/bench_$name.json; }
for r in 1 2; do
run qp_new_11m$r TGS_LIB=$L/libtidegs.so python bench.py --config 11m --moments persist --no-cpu-baseline --no-e2e --steps 200
run qp_old_11m$r TGS_LIB=$L/libtidegs_old.so python bench.py --config 11m --moments persist --no-cpu-baseline --no-e2e --steps 200
done
run qp_new_100m TGS_LIB=$L/libtidegs.so python bench.py --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 400 --steps 100
run qp_old_100m TGS_LIB=$L/libtidegs_old.so python bench.py --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 400 --steps 100
run qp_new_def TGS_LIB=$L/libtidegs.so python bench.py --no-cpu-baseline --no-e2e
rm -f $L/libtidegs_old.so
