# read-path shape on the GPU box's disk: runs of neighbouring misses, coalescing cap
mkdir -p gpurun_out
g++ -O2 -std=c++17 -pthread -I/usr/local/cuda/include -o /tmp/srb tools/store_readbench.cpp \
    paper_2605_20150_b200/csrc/tidegs_store.cpp -L/usr/local/cuda/lib64 -lcudart || exit 1
(
/tmp/srb /tmp/srb_store 30518 74 60 8 1 1 1
/tmp/srb /tmp/srb_store 30518 74 60 8 1 1 3
TGS_STORE_READ_RUN=1 /tmp/srb /tmp/srb_store 30518 74 60 8 1 1 3
/tmp/srb /tmp/srb_store 30518 74 60 8 1 1 8
TGS_STORE_READ_RUN=1 /tmp/srb /tmp/srb_store 30518 74 60 8 1 1 8
TGS_STORE_READ_RUN=1 /tmp/srb /tmp/srb_store 30518 74 60 16 1 1 8
) 2>&1 | grep -v "^base" | tee gpurun_out/srb3.txt
rm -rf /tmp/srb_store
