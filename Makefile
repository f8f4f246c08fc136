# Builds the product library (sm_100a) and the CPU oracle (test infrastructure).
#   paper_2312_10615_b200/libsmg.so  — C-ABI of include/smg.h (CUDA kernels + host driver)
#   oracle/liboracle.so              — CPU restatement used only by tests / baselines
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2312_10615_b200
CSRC := $(PKG)/csrc
# -fmad=false / -ffp-contract=off: no FMA contraction, so per-point arithmetic
# matches the oracle bit for bit.
NVFLAGS := $(ARCH) -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Xptxas -warn-spills
HOSTFLAGS := -O2 -std=c++17 -fPIC -ffp-contract=off -pthread -Wall -Wextra -I/usr/local/cuda/include

LIB := $(PKG)/libsmg.so
OBJS := build/kernels.o build/host.o

CLI := $(PKG)/solver

# test infrastructure: an NCCL stand-in that lets several ranks share one GPU (tests/test_gpu_zz_fake_ranks.py)
FAKE := tests/fake_nccl/libfakenccl.so

all: $(LIB) $(CLI) oracle $(FAKE)

# test infrastructure only: a failure here (e.g. no nccl.h) must not fail the product build; its tests skip
$(FAKE): tests/fake_nccl/fake_nccl.c
	-gcc -O2 -Wall -shared -fPIC -I/usr/local/cuda/include -o $@ $< -L/usr/local/cuda/lib64 -lcudart_static -lpthread -ldl -lrt

$(CLI): $(CSRC)/cli.cpp include/smg.h $(LIB)
	$(CXX) -O2 -std=c++17 -Wall -Wextra -o $@ $(CSRC)/cli.cpp -L$(PKG) -lsmg -Wl,-rpath,'$$ORIGIN'

build:
	mkdir -p build

build/kernels.o: $(CSRC)/kernels.cu $(CSRC)/smg_internal.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/host.o: $(CSRC)/host.cpp $(CSRC)/smg_internal.h include/smg.h | build
	$(CXX) $(HOSTFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -lpthread -ldl -lrt

oracle:
	$(MAKE) -s -C oracle

# tools-only instrumented library (per-warp phase timestamps; tools/trace_vanka.py)
trace: build/host.o | build
	$(NVCC) $(NVFLAGS) -DSMG_TRACE -c $(CSRC)/kernels.cu -o build/kernels_trace.o
	$(NVCC) $(ARCH) -shared -o tools/libsmg_trace.so build/kernels_trace.o build/host.o -lcudart_static -lpthread -ldl -lrt

clean:
	rm -rf build $(LIB) $(CLI) $(FAKE)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean trace
