# Builds the product library (CUDA, sm_100a) and the oracle (plain C, test infrastructure).
NVCC     ?= /usr/local/cuda/bin/nvcc
PKG      := paper_2411_01919_b200
SRC      := $(wildcard $(PKG)/csrc/*.cu)
CPPSRC   := $(wildcard $(PKG)/csrc/*.cpp)
OBJ      := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC)) $(patsubst $(PKG)/csrc/%.cpp,build/%.cpp.o,$(CPPSRC))
HDR      := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/pmap.h
LIB      := $(PKG)/libpmap.so
# --fmad=false: no implicit FMA contraction; every fused multiply-add the
# method prescribes is written as __fmaf_rn.
NVFLAGS  := -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
            -Xcompiler -fPIC,-fvisibility=hidden -Iinclude

all: $(LIB) oracle/liboracle.so

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $<

# host-only C++ (NEXT-4 map manager)
build/%.cpp.o: $(PKG)/csrc/%.cpp $(HDR)
	@mkdir -p build
	g++ -O2 -std=c++17 -fPIC -fvisibility=hidden -Iinclude -c -o $@ $<

$(LIB): $(OBJ)
	$(NVCC) -shared -gencode arch=compute_100a,code=sm_100a -o $@.tmp $(OBJ) && mv $@.tmp $@

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -std=c11 -fPIC -shared -ffp-contract=off -fno-fast-math -fvisibility=hidden -o $@ $< -lm

ptxas:
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/pmap_ptxas.o $(F) 2>&1 | grep -E "Function properties|registers|spill|smem|Compiling entry" | sed 's/ptxas info    ://'

clean:
	rm -rf $(LIB) oracle/liboracle.so build

.PHONY: all clean ptxas
