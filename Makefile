# Builds the three native libraries in-tree (they travel to the GPU box with gpurun):
#   paper_2605_10390_b200/libfractalsort.so  the product: C-ABI + sm_100a kernels
#   datagen/libfsdatagen.so                  seeded input generators (test/bench infrastructure)
#   oracle/liboracle.so                      the plain CPU oracle (test infrastructure)
NVCC      ?= nvcc
CC        ?= gcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Xptxas -v
CFLAGS    := -O2 -fPIC -Wall -Wextra -std=c11

PKG       := paper_2605_10390_b200
CSRC      := $(PKG)/csrc
KERNEL_SRCS := $(CSRC)/abi.cu $(CSRC)/hist16.cu $(CSRC)/scan.cu $(CSRC)/expand16.cu \
               $(CSRC)/wide.cu $(CSRC)/partition.cu $(CSRC)/host_stream.cu $(CSRC)/trie.cu $(CSRC)/peer.cu \
               $(CSRC)/small16.cu $(CSRC)/exchange.cu $(CSRC)/nvls.cu
KERNEL_HDRS := $(wildcard $(CSRC)/*.cuh) include/fractalsort.h
KERNEL_OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(KERNEL_SRCS))

all: $(PKG)/libfractalsort.so datagen/libfsdatagen.so oracle/liboracle.so

build/%.o: $(CSRC)/%.cu $(KERNEL_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Iinclude -dc -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libfractalsort.so: $(KERNEL_OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(KERNEL_OBJS)

datagen/libfsdatagen.so: datagen/datagen.cu datagen/fsg.h datagen/fsg_rng.h
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC -shared -o $@ datagen/datagen.cu

oracle/liboracle.so: oracle/oracle.c oracle/oracle_mt.c oracle/oracle.h
	$(CC) $(CFLAGS) -pthread -shared -o $@ oracle/oracle.c oracle/oracle_mt.c

clean:
	rm -rf build $(PKG)/libfractalsort.so datagen/libfsdatagen.so oracle/liboracle.so

.PHONY: all clean
