# steady-state timeline traces of two transfer splits; ncu k_adam / k_xfer capture
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name $(python tools/jline.py gpurun_out/bench_$name.json)"; }
TGS_TRACE=1 run trace_g8s4 --steps 12 --warmup 25 --no-cpu-baseline --no-e2e --no-persist-detail
grep "tgs trace" gpurun_out/bench_trace_g8s4.err | tail -120 > gpurun_out/trace_g8s4.txt
TGS_TRACE=1 TGS_GATHER_CTAS=8 TGS_SCATTER_CTAS=2 TGS_GATHER_BUFS=6 TGS_SCATTER_BUFS=6 run trace_g8s2 --steps 12 --warmup 25 --no-cpu-baseline --no-e2e --no-persist-detail
grep "tgs trace" gpurun_out/bench_trace_g8s2.err | tail -120 > gpurun_out/trace_g8s2.txt
B="python bench.py --steps 4 --warmup 26 --no-cpu-baseline --no-e2e --no-persist-detail"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_adam|k_xfer' -s 60 -c 4 -o gpurun_out/prof_r02 $B > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ncu -i gpurun_out/prof_r02.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw.csv 2>/dev/null; ls -la gpurun_out/ncu_full_raw.csv
