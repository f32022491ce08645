# Builds the sm_100a product library and the CPU checkers.
#   paper_1308_2400_b200/libafmm_b200.so   C ABI (include/afmm_b200.h) + CUDA kernels
#   oracle/liboracle.so, oracle/_ref/...    test infrastructure (see oracle/Makefile)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
           -Xptxas -warn-spills -Iinclude
# Bit-exactness: keep IEEE adds (no fast-math, no FTZ), no FMA contraction.
NVFLAGS += -fmad=false -ftz=false -prec-div=true -prec-sqrt=true

CSRC := paper_1308_2400_b200/csrc
SRCS := $(CSRC)/runtime.cu $(CSRC)/prepass.cu $(CSRC)/bform.cu $(CSRC)/peak.cu
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
LIB := paper_1308_2400_b200/libafmm_b200.so

all: $(LIB) oracle

build/%.o: $(CSRC)/%.cu $(CSRC)/common.cuh $(CSRC)/kernels.h include/afmm_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > build/libafmm_b200.sass

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean sass
