# Builds the sm_100a library in-tree (the .so travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xptxas -v -diag-suppress 1886 $(EXTRA)
SRC := $(wildcard paper_1912_02165_b200/csrc/*.cu)
HDR := $(wildcard paper_1912_02165_b200/csrc/*.cuh) include/winofuse_b200.h
OBJDIR := build
OBJ := $(patsubst paper_1912_02165_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))
LIB := paper_1912_02165_b200/libwinofuse_b200.so

all: $(LIB)

$(OBJDIR)/%.o: paper_1912_02165_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared $(OBJ) -o $@
	cat $(OBJDIR)/*.ptxas.log > build_ptxas.log

clean:
	rm -rf $(LIB) build_ptxas.log $(OBJDIR)

.PHONY: all clean
