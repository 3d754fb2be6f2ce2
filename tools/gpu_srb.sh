# host-only store read benchmark on the GPU box's disk (no GPU use)
mkdir -p gpurun_out
g++ -O2 -std=c++17 -pthread -o /tmp/srb tools/store_readbench.cpp paper_2605_20150_b200/csrc/tidegs_store.cpp || exit 1
for th in 8 16; do timeout 600 /tmp/srb /tmp/srb_store 30518 74 60 $th 1; done 2>&1 | tee gpurun_out/srb.txt
rm -rf /tmp/srb_store
