# Builds the CUDA hot path (libctis.so, sm_100a) and the CPU oracle (liboracle.so).
NVCC     ?= /usr/local/cuda/bin/nvcc
PKG      := paper_2006_01573_b200
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -Xptxas -v \
            --expt-relaxed-constexpr -Iinclude
SRCS     := $(PKG)/csrc/ctis_api.cu $(PKG)/csrc/ctis_kernels.cu
HDRS     := include/ctis.h $(PKG)/csrc/ctis_internal.h
OBJS     := $(patsubst %.cu,build/%.o,$(SRCS))

all: $(PKG)/libctis.so oracle/liboracle.so

build/%.o: %.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(PKG)/libctis.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -fPIC -o $@.tmp $(OBJS) && mv $@.tmp $@

oracle/liboracle.so: oracle/ctis_oracle.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -std=c99 -o $@ $<

clean:
	rm -rf build $(PKG)/libctis.so oracle/liboracle.so

.PHONY: all clean
