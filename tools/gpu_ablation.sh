# Ablations of the paper's T5 in this system's terms, 300m aerial, J=64.
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; tail -c 300 gpurun_out/bench_$name.json; echo; }
run abl_full --steps 30 --warmup 20
run abl_notide --no-tide --steps 10 --warmup 10
run abl_nooverlap --no-overlap --steps 30 --warmup 20
run abl_nomorton --config 300m_nomorton --fine-filter --steps 10 --warmup 10
run abl_refresh --refresh-bounds --steps 30 --warmup 20
