# Builds the product library (sm_100a only) and the CPU checkers under oracle/.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-Wall --expt-relaxed-constexpr
PKG       := paper_1610_10061_b200
CSRC      := $(wildcard $(PKG)/csrc/*.cu)
OBJS      := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))
LIB       := $(PKG)/libpmedian_b200.so

CLI       := $(PKG)/pmedian_bench

REFTESTS  := tests/cpp/_ref/ref_tests
REFACCEPT := tests/cpp/_ref/acceptance

all: $(LIB) $(CLI) oracle reftests

build/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/pmedian_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -warn-spills -c $< -o $@

# the scan (K2) schedules better with ptxas's aggressive register heuristics
# (syn20k 1.433 -> 1.415 ms, profiles/r02_k2_ab.md); the gather (gather.cu)
# does not (it loses occupancy), hence separate translation units
build/fitness.o: NVFLAGS += -Xptxas --register-usage-level=10
build_bounds/fitness.o: NVFLAGS += -Xptxas --register-usage-level=10

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -lrt -ldl -lpthread

# the reference CLI over the device path (host code; nvcc for the shared headers)
$(CLI): $(PKG)/cli/pmedian_bench.cpp $(LIB) $(PKG)/csrc/combinatorics.h
	$(NVCC) -x cu $(ARCH) -O2 -std=c++17 -o $@ $< -L$(PKG) -lpmedian_b200 -Xlinker -rpath,'$$ORIGIN'

oracle:
	$(MAKE) -s -C oracle

# Bounds-checked variant (-DPMB_BOUNDS: device PMB_CHECKs trap on an index outside
# its buffer); same sources, loaded with PMB_LIBRARY=$(BOUNDS_LIB) by
# tools/bounds_check.py and the GPU test suite.  Not part of `all`.
BOUNDS_OBJS := $(patsubst $(PKG)/csrc/%.cu,build_bounds/%.o,$(CSRC))
BOUNDS_LIB  := $(PKG)/libpmedian_b200_bounds.so
build_bounds/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/pmedian_b200.h
	@mkdir -p build_bounds
	$(NVCC) $(NVFLAGS) -DPMB_BOUNDS -c $< -o $@
$(BOUNDS_LIB): $(BOUNDS_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(BOUNDS_OBJS) -lcudart_static -lrt -ldl -lpthread
bounds: $(BOUNDS_LIB)

# TEST INFRASTRUCTURE: the reference's own unit tests (test_chromosome,
# test_instance, test_formulation, test_ga) compiled unchanged against the compat
# headers (include/compat/pmedian/ -> the device path) with a doctest stand-in.
# Built where /root/reference exists; the binary travels with the snapshot.
REF_TESTS_DIR ?= /root/reference/proj/tests
reftests: $(LIB)
	@if [ -d "$(REF_TESTS_DIR)" ]; then \
	  mkdir -p tests/cpp/_ref && \
	  g++ -std=c++20 -O1 -I include/compat -I include -I tests/cpp/doctest_shim tests/cpp/ref_tests_main.cpp \
	    $(REF_TESTS_DIR)/test_chromosome.cpp $(REF_TESTS_DIR)/test_instance.cpp $(REF_TESTS_DIR)/test_formulation.cpp \
	    $(REF_TESTS_DIR)/test_ga.cpp $(REF_TESTS_DIR)/test_bench.cpp $(REF_TESTS_DIR)/test_combinatorics.cpp \
	    -L $(PKG) -lpmedian_b200 -Wl,-rpath,'$$ORIGIN/../../../$(PKG)' -o $(REFTESTS).tmp && mv $(REFTESTS).tmp $(REFTESTS) && \
	  g++ -std=c++20 -O2 -I include/compat -I include $(REF_TESTS_DIR)/acceptance.cpp \
	    -L $(PKG) -lpmedian_b200 -Wl,-rpath,'$$ORIGIN/../../../$(PKG)' -o $(REFACCEPT).tmp && mv $(REFACCEPT).tmp $(REFACCEPT); \
	else echo "reftests: $(REF_TESTS_DIR) absent, keeping prebuilt $(REFTESTS) (if any)"; fi

clean:
	rm -rf build build_bounds $(LIB) $(BOUNDS_LIB) $(CLI)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle reftests clean bounds
