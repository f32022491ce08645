# Builds the sm_100a product library and the CPU checkers.
#   paper_1308_2400_b200/libafmm_b200.so   C ABI (include/afmm_b200.h) + CUDA kernels
#   oracle/liboracle.so, oracle/_ref/...    test infrastructure (see oracle/Makefile)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Xcompiler -mpclmul \
           -Xptxas -warn-spills -Iinclude
# Bit-exactness: keep IEEE adds (no fast-math, no FTZ), no FMA contraction.
NVFLAGS += -fmad=false -ftz=false -prec-div=true -prec-sqrt=true

CSRC := paper_1308_2400_b200/csrc
SRCS := $(CSRC)/runtime.cu $(CSRC)/prepass.cu $(CSRC)/bform.cu $(CSRC)/peak.cu $(CSRC)/generate.cu
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
LIB := paper_1308_2400_b200/libafmm_b200.so
REF_INC ?= /root/reference/proj/include

all: $(LIB) oracle $(if $(wildcard $(REF_INC)/afmm/kernels.hpp),cpptest)

build/%.o: $(CSRC)/%.cu $(CSRC)/common.cuh $(CSRC)/kernels.h $(CSRC)/costmodel.h \
           $(CSRC)/jumptable.inc $(CSRC)/mt64jump.h include/afmm_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle

# The reference's kernel tests restated against the drop-in C++ front end
# (needs the reference headers, so it is built in the build container; the
# binary travels to the GPU box with the snapshot).
cpptest: build/test_gpu_kernels build/afmm_gpu build/acceptance_gpu
build/afmm_gpu: tools/afmm_gpu_cli.cpp include/afmm_b200/kernels.hpp include/afmm_b200.h $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -ffp-contract=off -I$(REF_INC) -Iinclude -o $@ $< \
	    -L paper_1308_2400_b200 -lafmm_b200 -Wl,-rpath,'$$ORIGIN/../paper_1308_2400_b200'
build/test_gpu_kernels: tests/cpp/test_gpu_kernels.cpp include/afmm_b200/kernels.hpp include/afmm_b200.h $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -ffp-contract=off -I$(REF_INC) -Iinclude -o $@ $< \
	    -L paper_1308_2400_b200 -lafmm_b200 -Wl,-rpath,'$$ORIGIN/../paper_1308_2400_b200'

# The reference's acceptance gate with its AFMM calls on the B200 (test only)
build/acceptance_gpu: tests/cpp/acceptance_gpu.cpp tests/cpp/acceptance_gpu_shim.hpp include/afmm_b200/kernels.hpp include/afmm_b200.h $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -ffp-contract=off -I$(REF_INC) -Iinclude -Itests/cpp -o $@ $< \
	    -L paper_1308_2400_b200 -lafmm_b200 -Wl,-rpath,'$$ORIGIN/../paper_1308_2400_b200'

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > build/libafmm_b200.sass

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean sass cpptest checked

# Checked build (never the product): device bound checks counted into the
# call status + guard bands around every workspace buffer, verified after each
# product (compute-sanitizer is closed on this pool). Used by
# `AFMM_LIB=build/checked/libafmm_b200.so python tools/sanitize_cases.py`.
checked:
	@mkdir -p build/checked
	$(NVCC) $(NVFLAGS) -DAFMM_CHECKED -shared -o build/checked/libafmm_b200.so $(SRCS)

# Kernel timing experiments (never the product): build/exp/<name>/libafmm_b200.so
# with extra defines, selected at run time through AFMM_LIB.
exp-%:
	@mkdir -p build/exp/$*
	$(NVCC) $(NVFLAGS) $(EXPDEFS) -shared -o build/exp/$*/libafmm_b200.so $(SRCS)
