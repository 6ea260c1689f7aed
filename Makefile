# Build the in-tree CUDA library (sm_100a) and the oracle's C mirror.
# No --split-compile: it cuts the single translation unit's build from 6 to 2 minutes, but
# its partitioning changes the code generated for the same kernel source from build to
# build (the slab kernel came out in a 1408- and a 1864-instruction form, 28.9 vs 33.3 us).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           --expt-relaxed-constexpr -cudart static
LIBDIR := paper_2304_12168_b200/_lib
SRC := $(wildcard paper_2304_12168_b200/csrc/*.cu paper_2304_12168_b200/csrc/*.cuh) include/trisolve_b200.h

all: $(LIBDIR)/libtrisolve_b200.so

$(LIBDIR)/libtrisolve_b200.so: $(SRC)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -shared -o $@ paper_2304_12168_b200/csrc/ts_lib.cu

ptxas: $(SRC)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/ts_lib.o paper_2304_12168_b200/csrc/ts_lib.cu 2>&1 | grep -E "registers|spill|Compiling" | head -80

clean:
	rm -f $(LIBDIR)/*.so

.PHONY: all clean ptxas
