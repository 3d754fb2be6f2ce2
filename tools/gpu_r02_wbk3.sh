# write-back kernel shape (CTAs x buffers) under the copy-engine gather, same box
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/wbk3_$name.json 2> gpurun_out/wbk3_$name.err; echo "$name $(python tools/jline.py gpurun_out/wbk3_$name.json)"; }
for shape in "2 4" "2 3" "2 6" "3 3"; do
set -- $shape
TGS_WB_KERNEL=$1 TGS_SCATTER_BUFS=$2 run c$1b$2_w5 --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
TGS_WB_KERNEL=$1 TGS_SCATTER_BUFS=$2 run c$1b$2_w20 --no-cpu-baseline --no-persist-detail --no-e2e
done
