# copy-engine gather with the write-back as copy-engine runs (0), the TMA kernel with 1 CTA,
# 2 CTAs, or adaptive (-1: 1 CTA while the write-backs keep up, 4 when late); same box
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
TGS_WB_KERNEL=-1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "xfer or _ce" 2>&1 | tail -1
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/wbk_$name.json 2> gpurun_out/wbk_$name.err; echo "$name $(python tools/jline.py gpurun_out/wbk_$name.json)"; }
for r in 1 2; do
for v in 0 1 2 -1; do
TGS_WB_KERNEL=$v run v${v}_w5_$r --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
done
done
for v in 0 -1 1; do
TGS_WB_KERNEL=$v run v${v}_w20 --no-cpu-baseline --no-persist-detail --no-e2e
TGS_WB_KERNEL=$v run v${v}_100m --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
done
