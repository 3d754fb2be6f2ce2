mkdir -p gpurun_out
g++ -O2 -std=c++17 -pthread -I/usr/local/cuda/include -o /tmp/srb tools/store_readbench.cpp \
    paper_2605_20150_b200/csrc/tidegs_store.cpp -L/usr/local/cuda/lib64 -lcudart || exit 1
(
SRB_FILL=90 /tmp/srb /tmp/srb_store 30518 74 120 8 1 0 1 7887
SRB_FILL=90 /tmp/srb /tmp/srb_store 30518 74 120 8 1 1 1 7887
/tmp/srb /tmp/srb_store 30518 74 40 8 1 1 1 7887
/tmp/srb /tmp/srb_store 30518 74 40 8 1 1 1 2000
) 2>&1 | grep -v "^base" | tee gpurun_out/srb7.txt
cat /sys/kernel/mm/ksm/run 2>&1; cat /proc/sys/vm/overcommit_memory
rm -rf /tmp/srb_store
