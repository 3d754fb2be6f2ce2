# host store read benchmark on the GPU box's disk: pageable vs pinned cache, then the bench
mkdir -p gpurun_out
make -s || exit 1
g++ -O2 -std=c++17 -pthread -I/usr/local/cuda/include -o /tmp/srb tools/store_readbench.cpp \
    paper_2605_20150_b200/csrc/tidegs_store.cpp -L/usr/local/cuda/lib64 -lcudart || exit 1
for pin in 0 1; do timeout 600 /tmp/srb /tmp/srb_store 30518 74 60 8 1 $pin; done 2>&1 | tee gpurun_out/srb.txt
rm -rf /tmp/srb_store
timeout 900 python bench.py --config 1b --shard-of 8 --store /tmp/tgs_store --no-cpu-baseline --no-e2e > gpurun_out/bench_store1b_d.json 2> gpurun_out/bench_store1b_d.err
python tools/jline.py gpurun_out/bench_store1b_d.json
