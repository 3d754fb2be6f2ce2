mkdir -p gpurun_out
g++ -O2 -std=c++17 -pthread -I/usr/local/cuda/include -o /tmp/srb tools/store_readbench.cpp \
    paper_2605_20150_b200/csrc/tidegs_store.cpp -L/usr/local/cuda/lib64 -lcudart || exit 1
(
/tmp/srb /tmp/srb_store 30518 74 120 8 1 1 1 360
/tmp/srb /tmp/srb_store 30518 74 120 8 1 1 1 7887
/tmp/srb /tmp/srb_store 30518 74 120 8 1 0 1 7887
) 2>&1 | grep -v "^base" | tee gpurun_out/srb5.txt
rm -rf /tmp/srb_store
