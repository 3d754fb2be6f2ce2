# TGS_TRACE timelines of the default bench, copy-engine vs kernel transfers
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
for x in ce kernel; do
TGS_TRACE=1 timeout 900 python bench.py --xfer $x --steps 8 --warmup 25 --no-cpu-baseline --no-e2e --no-persist-detail > gpurun_out/trace_$x.json 2> gpurun_out/trace_$x.txt
python tools/jline.py gpurun_out/trace_$x.json
done
