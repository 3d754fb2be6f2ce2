# copy-engine transfer mode: parity of the affected tests, then a bench A/B (ce vs kernel)
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "xfer or ce or writeback or readmission or tide_off or small_pool or 300m or 1b" 2>&1 | tail -15 | tee gpurun_out/pytest_ce.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; tail -2 gpurun_out/bench_$name.err; }
run ce --xfer ce --no-cpu-baseline --no-persist-detail --steps 20 --warmup 5
run kernel --xfer kernel --no-cpu-baseline --no-persist-detail --steps 20 --warmup 5
run ce_long --xfer ce --no-cpu-baseline --no-persist-detail
run persist100_ce --config 100m --moments persist --xfer ce --no-cpu-baseline --warmup 100 --steps 100
