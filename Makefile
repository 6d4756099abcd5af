# Build everything in-tree (the .so files travel to the GPU box with gpurun).
#   make            -> paper_1305_3345_b200/libkgpu.so, oracle/libkgo.so, build/test_kat, build/pipes
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xptxas -v
PKG     := paper_1305_3345_b200
CSRC    := $(PKG)/csrc
LIB     := $(PKG)/libkgpu.so

all: $(LIB) oracle/libkgo.so build/test_kat build/pipes build/latency build/kgpu_crypt build/e1

build:
	mkdir -p build

build/%.o: $(CSRC)/%.cu $(CSRC)/kg_internal.h $(wildcard $(CSRC)/*.cuh) include/kg.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

build/%.o: $(CSRC)/%.cpp $(CSRC)/kg_internal.h include/kg.h | build
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

$(LIB): build/kg_kernels.o build/kg_tables.o build/kg_runtime.o
	$(NVCC) $(ARCH) -shared -cudart static -o $@.tmp $^ -Xcompiler -fvisibility=hidden && mv $@.tmp $@

# ORACLE (test infrastructure; never linked into the product)
oracle/libkgo.so: oracle/kgo_aes.c oracle/kgo_pages.c oracle/kgo_aes.h
	gcc -std=c99 -O2 -fPIC -shared -D_POSIX_C_SOURCE=200809L -Wall -o $@ oracle/kgo_aes.c oracle/kgo_pages.c -lpthread

build/test_kat: oracle/kgo_aes.c oracle/kgo_pages.c oracle/test_kat.c oracle/kgo_aes.h | build
	gcc -std=c99 -O2 -D_POSIX_C_SOURCE=200809L -Wall -o $@ oracle/kgo_aes.c oracle/kgo_pages.c oracle/test_kat.c -lpthread

# pipe microbenchmarks (roofline inputs)
build/pipes: tools/pipes.cu | build
	$(NVCC) -O3 -lineinfo -std=c++17 $(ARCH) -o $@ $<

build/latency: tools/latency.cu include/kg.h $(LIB) | build
	$(NVCC) -O2 -std=c++17 $(ARCH) -Iinclude -o $@ $< -L$(PKG) -lkgpu -Xlinker -rpath,'$$ORIGIN/../$(PKG)'

# the paper's §3.1 E1 experiment: launch vs CUDA graph vs persistent kernel at 512/1024/2048 threads
build/e1: tools/e1.cu | build
	$(NVCC) -O2 -std=c++17 $(ARCH) -o $@ $<

build/kgpu_crypt: examples/kgpu_crypt.c include/kg.h $(LIB) | build
	gcc -std=c99 -O2 -Wall -Iinclude -o $@ $< -L$(PKG) -lkgpu -Wl,-rpath,'$$ORIGIN/../$(PKG)'

# diagnostics (not part of `all`): copy-engine overlap, per-CTA stamps, bitsliced round
tools: build/zc_duplex build/bitslice_bp build/copy_overlap build/cta_stamps build/bitslice_bench build/soak_tsan build/pipes_tex build/pipes_lds build/pipes_ldpath \
       build/hybrid_bench build/hybrid_throttle build/pipe_variants

build/zc_duplex: tools/zc_duplex.cu | build
	$(NVCC) -O2 -std=c++17 $(ARCH) -o $@ $<

build/bitslice_bp: tools/bitslice_bp.cu tools/kg_sbox_bp.cuh tools/kg_sbox_bs.cuh | build
	$(NVCC) -O3 -std=c++17 $(ARCH) -Itools -o $@ $<

build/copy_overlap: tools/copy_overlap.cu | build
	$(NVCC) -O2 $(ARCH) -o $@ $<

build/cta_stamps: tools/cta_stamps.cu $(CSRC)/kg_kernels.cu $(CSRC)/kg_tables.cpp $(wildcard $(CSRC)/*.cuh) | build
	$(NVCC) -O3 -std=c++17 $(ARCH) -o $@ $< $(CSRC)/kg_tables.cpp

build/pipes_tex build/pipes_lds build/pipes_ldpath: build/%: tools/%.cu | build
	$(NVCC) -O3 -std=c++17 $(ARCH) -o $@ $<

build/hybrid_bench: tools/hybrid_bench.cu tools/kg_sbox_bs.cuh | build
	$(NVCC) -O3 -std=c++17 $(ARCH) -Itools -o $@ $<

build/hybrid_throttle: tools/hybrid_throttle.cu tools/kg_sbox_bp.cuh | build
	$(NVCC) -O3 -std=c++17 $(ARCH) -Itools -o $@ $<

build/pipe_variants: tools/pipe_variants.cu | build
	$(NVCC) -O2 -std=c++17 $(ARCH) -o $@ $< -lcuda

build/bitslice_bench: tools/bitslice_bench.cu tools/kg_sbox_bs.cuh | build
	$(NVCC) -O3 -std=c++17 $(ARCH) -o $@ $<

# host runtime under ThreadSanitizer (kernels unchanged; kg_runtime.cpp + kg_tables.cpp instrumented)
build/soak_tsan: tools/soak_tsan.cpp $(CSRC)/kg_runtime.cpp $(CSRC)/kg_tables.cpp build/kg_kernels.o | build
	g++ -std=c++17 -O1 -g -fsanitize=thread -Iinclude -I/usr/local/cuda/include -c $(CSRC)/kg_runtime.cpp -o build/kg_runtime_tsan.o
	g++ -std=c++17 -O1 -g -fsanitize=thread -I/usr/local/cuda/include -c $(CSRC)/kg_tables.cpp -o build/kg_tables_tsan.o
	$(NVCC) $(ARCH) -o $@ tools/soak_tsan.cpp build/kg_runtime_tsan.o build/kg_tables_tsan.o build/kg_kernels.o \
	  -Iinclude -Xcompiler -fsanitize=thread -ltsan -lpthread

# bounds-checked library (KG_BOUNDS_CHECK: every global page/IV/key-id access checked, trap on a
# violation; stands in for compute-sanitizer memcheck): KG_LIBKGPU=build/bounds/libkgpu_bounds.so
bounds: build/bounds/libkgpu_bounds.so

build/bounds/libkgpu_bounds.so: $(CSRC)/kg_kernels.cu $(CSRC)/kg_tables.cpp $(CSRC)/kg_runtime.cpp $(CSRC)/kg_internal.h $(wildcard $(CSRC)/*.cuh) include/kg.h
	mkdir -p build/bounds
	$(NVCC) $(NVFLAGS) -DKG_BOUNDS_CHECK -c $(CSRC)/kg_kernels.cu -o build/bounds/kg_kernels.o 2> build/bounds/kg_kernels.ptxas.txt || (cat build/bounds/kg_kernels.ptxas.txt; false)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ build/bounds/kg_kernels.o build/kg_tables.o build/kg_runtime.o -Xcompiler -fvisibility=hidden

clean:
	rm -rf build $(LIB) oracle/libkgo.so

.PHONY: all clean tools bounds
