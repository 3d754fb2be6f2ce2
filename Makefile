# Builds every native artefact in-tree (the .so files travel to the GPU box
# with the gpurun snapshot).  CUDA code targets sm_100a only.
NVCC      ?= /usr/local/cuda/bin/nvcc
CUDA_ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -lineinfo -std=c++17 $(CUDA_ARCH) -Xcompiler -fPIC -Xcompiler -fno-fast-math \
             -Xcompiler -ffp-contract=off -cudart static -Xptxas -v
PKG       := paper_2605_20150_b200

PRODUCT   := $(if $(wildcard $(PKG)/csrc/tidegs_kernels.cu),$(PKG)/libtidegs.so,)

all: workload/libtgsworkload.so workload/libtgsworkload_cuda.so oracle/libtgsoracle.so $(PRODUCT)

# seeded input generators (shared by both sides; no method arithmetic)
workload/libtgsworkload.so: workload/tgs_workload.c workload/tgs_workload.h
	gcc -O2 -fPIC -shared -ffp-contract=off -fno-fast-math -o $@ $< -lm -lpthread

workload/libtgsworkload_cuda.so: workload/tgs_workload_cuda.cu
	$(NVCC) $(NVFLAGS) -shared -o $@ $< 2> workload/ptxas_workload.log || (cat workload/ptxas_workload.log; false)

# the oracle: plain single-threaded C++17, no FMA contraction, no fast-math
oracle/libtgsoracle.so: oracle/tgs_oracle.cpp oracle/tgs_oracle.h
	g++ -std=c++17 -O2 -fPIC -shared -ffp-contract=off -fno-fast-math -o $@ $<

# the product: CUDA kernels + C++ runtime behind the C ABI (include/tidegs.h)
$(PKG)/libtidegs.so: $(PKG)/csrc/tidegs_kernels.cu $(PKG)/csrc/tidegs_runtime.cu \
                     $(PKG)/csrc/tidegs_store.cpp $(PKG)/csrc/tidegs_store.h \
                     $(PKG)/csrc/tidegs_order.cu \
                     $(PKG)/csrc/tidegs_internal.h include/tidegs.h
	$(NVCC) $(NVFLAGS) -Iinclude -shared -o $@ $(PKG)/csrc/tidegs_kernels.cu \
	    $(PKG)/csrc/tidegs_runtime.cu $(PKG)/csrc/tidegs_store.cpp $(PKG)/csrc/tidegs_order.cu \
	    -lpthread 2> $(PKG)/ptxas.log || (cat $(PKG)/ptxas.log; false)

clean:
	rm -f workload/*.so oracle/*.so $(PKG)/*.so

.PHONY: all clean
