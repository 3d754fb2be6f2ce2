# span traces of the compute-bound regimes (100m persist; the whole 1B shard resident)
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
TGS_TRACE=1 timeout 900 python bench.py --config 100m --moments persist --steps 6 --warmup 400 --no-cpu-baseline --no-e2e > gpurun_out/trace_100m.json 2> gpurun_out/trace_100m.txt
python tools/jline.py gpurun_out/trace_100m.json
TGS_TRACE=1 timeout 900 python bench.py --config 1b --shard-of 8 --capacity 244141 --pool-slots 30518 --steps 6 --warmup 100 --no-cpu-baseline --no-e2e > gpurun_out/trace_1binf.json 2> gpurun_out/trace_1binf.txt
python tools/jline.py gpurun_out/trace_1binf.json
