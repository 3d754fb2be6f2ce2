# k_xfer bring-up: smoke, GPU tests (incl. the new full-size capacity-bound ones),
# default bench and a gather/scatter CTA sweep.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.log
timeout 2700 python -m pytest tests -m gpu -x -q --durations=15 2>&1 | tail -30 | tee gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; python tools/jline.py gpurun_out/bench_$name.json; tail -2 gpurun_out/bench_$name.err; }
run default --steps 20 --warmup 5
for gc in 4 8 16; do for sc in 2 4 8; do
  TGS_GATHER_CTAS=$gc TGS_SCATTER_CTAS=$sc run sweep_g${gc}_s${sc} --steps 30 --warmup 20 --no-cpu-baseline --no-e2e
done; done
