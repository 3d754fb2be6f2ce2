# write-back kernel shapes under the copy-engine gather, round 2 (same box)
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/wbk_$name.json 2> gpurun_out/wbk_$name.err; echo "$name $(python tools/jline.py gpurun_out/wbk_$name.json)"; }
for v in 0 2 -2 3; do
TGS_WB_KERNEL=$v run b${v}_w5 --no-cpu-baseline --no-persist-detail --no-e2e --steps 20 --warmup 5
TGS_WB_KERNEL=$v run b${v}_w20 --no-cpu-baseline --no-persist-detail --no-e2e
TGS_WB_KERNEL=$v run b${v}_100m --config 100m --moments persist --no-cpu-baseline --no-e2e --warmup 100 --steps 100
done
