# Builds the CUDA hot path (libctis.so, sm_100a) and the CPU oracle (liboracle.so).
NVCC     ?= /usr/local/cuda/bin/nvcc
PKG      := paper_2006_01573_b200
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
            --expt-relaxed-constexpr -Iinclude -Ibuild
HDRS     := include/ctis.h $(PKG)/csrc/ctis_internal.h $(PKG)/csrc/ctis_kernels.h $(PKG)/csrc/ctis_fft.h \
            $(PKG)/csrc/ctis_comm.h
# nccl.h for the latency mode's types (the library itself is dlopen'ed at run time)
NCCL_INC ?= $(shell python -c "import os, nvidia.nccl as m; print(os.path.join(list(m.__path__)[0], 'include'))" 2>/dev/null || echo /usr/include)

all: $(PKG)/libctis.so oracle/liboracle.so

# Projection kernels: a standalone cubin, embedded and loaded once per plan tap page.
build/ctis_tables.cubin: $(PKG)/csrc/ctis_tables.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Iinclude -cubin -Xptxas -v $< -o $@ 2> build/ctis_tables.ptxas.log \
	  || (cat build/ctis_tables.ptxas.log; false)

# embedded with .incbin (assembling a 10 MB array literal through nvcc takes minutes)
build/ctis_tables_blob.o: build/ctis_tables.cubin
	printf '.section .rodata\n.balign 16\n.globl ctis_tables_cubin\n.globl ctis_tables_cubin_end\n.hidden ctis_tables_cubin\n.hidden ctis_tables_cubin_end\nctis_tables_cubin:\n.incbin "%s"\nctis_tables_cubin_end:\n.byte 0\n.section .note.GNU-stack,"",@progbits\n' $(abspath $<) > build/ctis_tables_blob.S
	gcc -c build/ctis_tables_blob.S -o $@

build/ctis_api.o: $(PKG)/csrc/ctis_api.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/ctis_comm.o: $(PKG)/csrc/ctis_comm.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -I$(NCCL_INC) -c $< -o $@

build/ctis_fft.o: $(PKG)/csrc/ctis_fft.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/ctis_kernels.o: $(PKG)/csrc/ctis_kernels.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/ctis_kernels.ptxas.log || (cat build/ctis_kernels.ptxas.log; false)

$(PKG)/libctis.so: build/ctis_api.o build/ctis_kernels.o build/ctis_fft.o build/ctis_comm.o build/ctis_tables_blob.o
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -fPIC -o $@.tmp $^ -lcufft -ldl && mv $@.tmp $@

oracle/liboracle.so: oracle/ctis_oracle.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -std=c99 -o $@ $<

build/microbench: tools/microbench.cu
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 -o $@ $<

clean:
	rm -rf build $(PKG)/libctis.so oracle/liboracle.so

.PHONY: all clean
