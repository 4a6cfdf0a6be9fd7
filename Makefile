# Builds the sm_100a library in-tree (the .so travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xptxas -v -diag-suppress 1886 $(EXTRA)
SRC := $(wildcard paper_1912_02165_b200/csrc/*.cu)
HDR := $(wildcard paper_1912_02165_b200/csrc/*.cuh) include/winofuse_b200.h
LIB := paper_1912_02165_b200/libwinofuse_b200.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared $(SRC) -o $@ 2> build_ptxas.log || (cat build_ptxas.log; false)

clean:
	rm -f $(LIB) build_ptxas.log

.PHONY: all clean
