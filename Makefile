# Builds the product library (CUDA kernels + C-ABI) for sm_100a, in-tree, and
# the test-only checkers under oracle/.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O2,-ffp-contract=off
SRC := paper_1712_03439_b200/csrc
OUT := paper_1712_03439_b200/_lib
OBJS := $(OUT)/kernels.o $(OUT)/api.o

all: $(OUT)/libroomsim_gpu.so oracle

$(OUT)/kernels.o: $(SRC)/kernels.cu $(SRC)/kernels.cuh $(SRC)/fft.cuh
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OUT)/kernels.ptxas.log || (cat $(OUT)/kernels.ptxas.log; false)

$(OUT)/api.o: $(SRC)/api.cu $(SRC)/kernels.cuh include/roomsim_gpu.h
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OUT)/libroomsim_gpu.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf $(OUT)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
