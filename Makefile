# Builds the CUDA hot path (libctis.so, sm_100a) and the CPU oracle (liboracle.so).
NVCC     ?= /usr/local/cuda/bin/nvcc
PKG      := paper_2006_01573_b200
ARCH     := -gencode arch=compute_100a,code=sm_100a
# experiment builds: make BUILD=build_x EXTRA='-DFOO=1' LIBOUT=build_x/libctis.so (CTIS_LIB_PATH selects it)
BUILD    ?= build
EXTRA    ?=
LIBOUT   ?= $(PKG)/libctis.so
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
            --expt-relaxed-constexpr -Iinclude $(EXTRA)
HDRS     := include/ctis.h $(PKG)/csrc/ctis_internal.h $(PKG)/csrc/ctis_strip_dispatch.inc $(PKG)/csrc/ctis_kernels.h $(PKG)/csrc/ctis_fft.h \
            $(PKG)/csrc/ctis_comm.h $(PKG)/csrc/ctis_nvls.h
# nccl.h for the latency mode's types (the library itself is dlopen'ed at run time)
NCCL_INC ?= $(shell python -c "import os, nvidia.nccl as m; print(os.path.join(list(m.__path__)[0], 'include'))" 2>/dev/null || echo /usr/include)

all: $(LIBOUT) oracle/liboracle.so

# Projection kernels: a standalone cubin, embedded and loaded once per plan tap page.
$(BUILD)/ctis_tables.cubin: $(PKG)/csrc/ctis_tables.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Iinclude $(EXTRA) -cubin -Xptxas -v $< -o $@ 2> $(BUILD)/ctis_tables.ptxas.log \
	  || (cat $(BUILD)/ctis_tables.ptxas.log; false)

# embedded with .incbin (assembling a 10 MB array literal through nvcc takes minutes)
$(BUILD)/ctis_tables_blob.o: $(BUILD)/ctis_tables.cubin
	printf '.section .rodata\n.balign 16\n.globl ctis_tables_cubin\n.globl ctis_tables_cubin_end\n.hidden ctis_tables_cubin\n.hidden ctis_tables_cubin_end\nctis_tables_cubin:\n.incbin "%s"\nctis_tables_cubin_end:\n.byte 0\n.section .note.GNU-stack,"",@progbits\n' $(abspath $<) > $(BUILD)/ctis_tables_blob.S
	gcc -c $(BUILD)/ctis_tables_blob.S -o $@

$(BUILD)/ctis_api.o: $(PKG)/csrc/ctis_api.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/ctis_comm.o: $(PKG)/csrc/ctis_comm.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -I$(NCCL_INC) -c $< -o $@

# the fused NVLink exchange kernel uses NCCL's device API (header-only device code, nccl_device.h)
$(BUILD)/ctis_nvls.o: $(PKG)/csrc/ctis_nvls.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -I$(NCCL_INC) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ctis_nvls.ptxas.log || (cat $(BUILD)/ctis_nvls.ptxas.log; false)

$(BUILD)/ctis_fft.o: $(PKG)/csrc/ctis_fft.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/ctis_kernels.o: $(PKG)/csrc/ctis_kernels.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ctis_kernels.ptxas.log || (cat $(BUILD)/ctis_kernels.ptxas.log; false)

$(LIBOUT): $(BUILD)/ctis_api.o $(BUILD)/ctis_kernels.o $(BUILD)/ctis_fft.o $(BUILD)/ctis_comm.o $(BUILD)/ctis_nvls.o \
          $(BUILD)/ctis_tables_blob.o
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -fPIC -o $@.tmp $^ -lcufft -ldl && mv $@.tmp $@

oracle/liboracle.so: oracle/ctis_oracle.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -std=c99 -o $@ $<

$(BUILD)/microbench: tools/microbench.cu
	@mkdir -p $(BUILD)
	$(NVCC) $(ARCH) -O3 -o $@ $<

clean:
	rm -rf $(BUILD) $(LIBOUT) oracle/liboracle.so

.PHONY: all clean
