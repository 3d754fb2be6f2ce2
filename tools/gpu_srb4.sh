# is the bench's own base segment slow to read (file layout), or the bench process?
mkdir -p gpurun_out
make -s || exit 1
TGS_KEEP_STORE=1 timeout 900 python bench.py --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/bench_store1b_e.json 2> gpurun_out/bench_store1b_e.err
python tools/jline.py gpurun_out/bench_store1b_e.json
ls -la /tmp/tgs_store/rank000 | head; filefrag /tmp/tgs_store/rank000/base.tdgs 2>&1 | tail -1
timeout 300 python tools/ssd_probe.py /tmp/tgs_store/rank000/base.tdgs 966656 2>&1 | tee gpurun_out/ssd_probe_benchfile.txt
rm -rf /tmp/tgs_store
