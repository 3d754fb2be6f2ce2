# copy-engine run copies over one vs two streams per direction (TGS_CE_STREAMS), same box
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
TGS_CE_STREAMS=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "xfer or _ce" 2>&1 | tail -1
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/ces_$name.json 2> gpurun_out/ces_$name.err; echo "$name $(python tools/jline.py gpurun_out/ces_$name.json)"; }
for r in 1 2 3; do
TGS_CE_STREAMS=2 run s2_w5_$r --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
TGS_CE_STREAMS=1 run s1_w5_$r --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
done
TGS_CE_STREAMS=2 run s2_100m --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
TGS_CE_STREAMS=1 run s1_100m --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
