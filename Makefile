# Build everything in-tree (the .so files travel to the GPU box with gpurun).
#   make            -> paper_2101_11714_b200/lib/libttgpu.so  (sm_100a, product)
#                      oracle/libttoracle.so, oracle/_ref/libttref.so (test infra)
NVCC     ?= nvcc
PKG      := paper_2101_11714_b200
CSRC     := $(PKG)/csrc
LIB      := $(PKG)/lib/libttgpu.so
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -std=c++17 -O3 -lineinfo $(ARCH) -Xcompiler -fPIC -shared -Xptxas -v
SRCS     := $(CSRC)/ttgpu.cu $(CSRC)/shape_plan.cpp
HDRS     := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp) $(wildcard $(CSRC)/*.inl) include/ttgpu.h

DIAG     := $(PKG)/lib/libttgpu_diag.so

.PHONY: all lib lib-diag oracle clean
all: lib oracle

lib: $(LIB)

# diagnostics build: per-CTA timelines (bench.py --cta-times, TTGPU_LIB=$(DIAG))
lib-diag: $(DIAG)

$(DIAG): $(SRCS) $(HDRS)
	mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -DTTGPU_CTA_TIMES -o $@ $(SRCS) 2> $(PKG)/lib/ptxas_diag.log || (cat $(PKG)/lib/ptxas_diag.log; false)

$(LIB): $(SRCS) $(HDRS)
	mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -o $@ $(SRCS) 2> $(PKG)/lib/ptxas.log || (cat $(PKG)/lib/ptxas.log; false)

oracle:
	$(MAKE) -C oracle all

clean:
	rm -f $(LIB) $(DIAG)
	$(MAKE) -C oracle clean
