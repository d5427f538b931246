# Builds the product library (sm_100a only) and the CPU checkers under oracle/.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-Wall --expt-relaxed-constexpr
PKG       := paper_1610_10061_b200
CSRC      := $(wildcard $(PKG)/csrc/*.cu)
OBJS      := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))
LIB       := $(PKG)/libpmedian_b200.so

all: $(LIB) oracle

build/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/pmedian_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -warn-spills -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -lrt -ldl -lpthread

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean
