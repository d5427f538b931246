# Builds the product library (sm_100a only) and the CPU checkers under oracle/.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-Wall --expt-relaxed-constexpr
PKG       := paper_1610_10061_b200
CSRC      := $(wildcard $(PKG)/csrc/*.cu)
OBJS      := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))
LIB       := $(PKG)/libpmedian_b200.so

CLI       := $(PKG)/pmedian_bench

all: $(LIB) $(CLI) oracle

build/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/pmedian_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -warn-spills -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -lrt -ldl -lpthread

# the reference CLI over the device path (host code; nvcc for the shared headers)
$(CLI): $(PKG)/cli/pmedian_bench.cpp $(LIB) $(PKG)/csrc/combinatorics.h
	$(NVCC) -x cu $(ARCH) -O2 -std=c++17 -o $@ $< -L$(PKG) -lpmedian_b200 -Xlinker -rpath,'$$ORIGIN'

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB) $(CLI)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean
