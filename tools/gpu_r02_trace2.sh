set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
TGS_TRACE=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-persist-detail > gpurun_out/trace_cm.json 2> gpurun_out/trace_cm.txt
python tools/jline.py gpurun_out/trace_cm.json
