# Builds the product library (CUDA kernels + C-ABI) for sm_100a, in-tree, and
# the test-only checkers under oracle/.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
EXTRA ?=
NVFLAGS := $(ARCH) $(EXTRA) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O2,-ffp-contract=off
SRC := paper_1712_03439_b200/csrc
OUT := paper_1712_03439_b200/_lib
OBJS := $(OUT)/kernels.o $(OUT)/big.o $(OUT)/large.o $(OUT)/ola2.o $(OUT)/synth_bound.o $(OUT)/sampler.o $(OUT)/features.o $(OUT)/api.o

REF_INC ?= /root/reference/proj/include
ADAPTER := tests/cpp/_build/adapter_test

all: $(OUT)/libroomsim_gpu.so oracle adapter

$(OUT)/kernels.o: $(SRC)/kernels.cu $(SRC)/kernels.cuh $(SRC)/mixfin.cuh $(SRC)/power.cuh $(SRC)/fft.cuh $(SRC)/async.cuh
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OUT)/kernels.ptxas.log || (cat $(OUT)/kernels.ptxas.log; false)

$(OUT)/large.o: $(SRC)/large.cu $(SRC)/kernels.cuh $(SRC)/power.cuh $(SRC)/fft.cuh $(SRC)/async.cuh
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OUT)/large.ptxas.log || (cat $(OUT)/large.ptxas.log; false)

$(OUT)/big.o: $(SRC)/big.cu $(SRC)/kernels.cuh $(SRC)/mixfin.cuh $(SRC)/power.cuh $(SRC)/fft.cuh
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OUT)/big.ptxas.log || (cat $(OUT)/big.ptxas.log; false)

$(OUT)/ola2.o: $(SRC)/ola2.cu $(SRC)/kernels.cuh $(SRC)/power.cuh $(SRC)/fft.cuh $(SRC)/fft2.cuh $(SRC)/async.cuh
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OUT)/ola2.ptxas.log || (cat $(OUT)/ola2.ptxas.log; false)

$(OUT)/synth_bound.o: $(SRC)/synth_bound.cu $(SRC)/kernels.cuh
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OUT)/synth_bound.ptxas.log || (cat $(OUT)/synth_bound.ptxas.log; false)

$(OUT)/sampler.o: $(SRC)/sampler.cu $(SRC)/sampler.cuh include/roomsim_gpu.h
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OUT)/features.o: $(SRC)/features.cu $(SRC)/kernels.cuh $(SRC)/mixfin.cuh $(SRC)/power.cuh $(SRC)/fft.cuh
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OUT)/api.o: $(SRC)/api.cu $(SRC)/kernels.cuh $(SRC)/mixfin.cuh $(SRC)/power.cuh include/roomsim_gpu.h
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -Xcompiler -fopenmp -c $< -o $@

$(OUT)/libroomsim_gpu.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -lgomp -ldl

oracle:
	$(MAKE) -s -C oracle

# C++ drop-in test against the reference headers (only where they exist; the
# binary travels to the GPU box like the .so files).
adapter: $(OUT)/libroomsim_gpu.so
	@if [ -d "$(REF_INC)/roomsim" ]; then \
	  mkdir -p tests/cpp/_build && \
	  g++ -O2 -std=c++20 -I$(REF_INC) -Iinclude -I/usr/local/cuda/include tests/cpp/adapter_test.cpp \
	    -L$(OUT) -lroomsim_gpu -Wl,-rpath,'$$ORIGIN/../../../$(OUT)' -o $(ADAPTER); \
	else echo "reference headers not present; keeping prebuilt $(ADAPTER) (if any)"; fi

clean:
	rm -rf $(OUT)
	$(MAKE) -C oracle clean

.PHONY: all oracle adapter clean
