# Build recipe for the B200-native PBD-R library (invoked by __graft_entry__.build()).
#
#   make            -> paper_2603_14634_b200/lib/libpbdr_gpu.so  (product: sm_100a CUDA + C-ABI)
#                      oracle/build/liboracle.so                (test infrastructure)
#                      build/test_dropin                        (C++ drop-in API test driver)
#   make ref        -> oracle/_ref/libpbdr_ref.so (needs /root/reference; this container only)
#
# --fmad=false keeps every fp32/fp64 product and sum separately rounded, which
# is what lets the CUDA path reproduce the CPU oracle bit for bit.

NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      := /usr/bin/g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2603_14634_b200
CSRC     := $(PKG)/csrc
LIB      := $(PKG)/lib/libpbdr_gpu.so
# Host-only half (scene generation, RNG, pack_box, the thread-local error
# state): no CUDA, so the CPU reference arm of bench.py can build its inputs
# without mapping the GPU library. libpbdr_gpu.so links against it.
HOST_LIB := $(PKG)/lib/libpbdr_host.so
NVFLAGS  := $(ARCH) -std=c++17 -O3 -lineinfo --fmad=false -Xcompiler -fPIC,-ffp-contract=off \
            -Xptxas -v -Iinclude -I$(CSRC)
CU_SRC   := $(CSRC)/pbdr_kernels.cu $(CSRC)/pbdr_sort.cu $(CSRC)/pbdr_engine.cu $(CSRC)/pbdr_mesh.cu \
            $(CSRC)/pbdr_slab.cu
CXX_SRC  := $(CSRC)/pbdr_dropin.cpp
HOST_SRC := $(CSRC)/pbdr_scene.cpp $(CSRC)/pbdr_errors.cpp $(CSRC)/pbdr_hostmath.cpp $(CSRC)/pbdr_body.cpp
HDRS     := include/pbdr_gpu.h $(wildcard include/pbdr/*.hpp) $(wildcard $(CSRC)/*.h) $(wildcard $(CSRC)/*.cuh)
OBJDIR   := build/obj
CU_OBJ   := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRC))
CXX_OBJ  := $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.o,$(CXX_SRC))
HOST_OBJ := $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.o,$(HOST_SRC))

.PHONY: all lib oracle ref clean checked
all: lib oracle build/test_dropin build/libdropin_shim.so checked

lib: $(HOST_LIB) $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.txt || (cat $(OBJDIR)/$*.ptxas.txt; false)

$(OBJDIR)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX) -std=c++17 -O3 -fPIC -ffp-contract=off -Wall -Wextra -Iinclude -I$(CSRC) \
	    -I/usr/local/cuda/include -c $< -o $@

$(HOST_LIB): $(HOST_OBJ)
	@mkdir -p $(PKG)/lib
	$(CXX) -shared -o $@ $^

$(LIB): $(CU_OBJ) $(CXX_OBJ) $(HOST_LIB)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJ) $(CXX_OBJ) -L$(PKG)/lib -lpbdr_host -lcudart -lnccl \
	    -Xlinker -rpath,'$$ORIGIN'

# Checked build: the same library with device-side bounds / invariant checks
# (PBDR_CHECKED, csrc/pbdr_kernels.cu). Run the GPU tests against it with
# PBDR_LIB_PATH=$(PWD)/paper_2603_14634_b200/lib/libpbdr_gpu_checked.so.
CHECKED  := $(PKG)/lib/libpbdr_gpu_checked.so
checked: $(CHECKED)
$(OBJDIR)/checked/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)/checked
	$(NVCC) $(NVFLAGS) -DPBDR_CHECKED=1 -c $< -o $@ 2> $(OBJDIR)/checked/$*.ptxas.txt || (cat $(OBJDIR)/checked/$*.ptxas.txt; false)
$(CHECKED): $(patsubst $(CSRC)/%.cu,$(OBJDIR)/checked/%.o,$(CU_SRC)) $(CXX_OBJ) $(HOST_LIB)
	$(NVCC) $(ARCH) -shared -o $@ $(patsubst $(CSRC)/%.cu,$(OBJDIR)/checked/%.o,$(CU_SRC)) $(CXX_OBJ) \
	    -L$(PKG)/lib -lpbdr_host -lcudart -lnccl -Xlinker -rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle

ref:
	$(MAKE) -C oracle ref

build/test_dropin: tests/cpp/test_dropin.cpp $(LIB) $(HDRS)
	@mkdir -p build
	$(CXX) -std=c++17 -O2 -Iinclude tests/cpp/test_dropin.cpp -o $@ \
	    -L$(PKG)/lib -lpbdr_gpu -lpbdr_host -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib'

# Test infrastructure: the oracle's extern "C" shim over the reference's public
# math/body/geometry API (oracle/ref_shim.cpp), compiled UNCHANGED against this
# repository's drop-in headers (include/pbdr/*.hpp) and libraries instead of the
# reference's. tests/test_dropin_headers.py compares it with the same shim
# built on the reference's own code (oracle/_ref/libpbdr_ref.so).
build/libdropin_shim.so: oracle/ref_shim.cpp $(HOST_LIB) $(LIB) $(HDRS)
	@mkdir -p build
	$(CXX) -std=c++20 -O2 -fPIC -shared -Wall -Wextra -Iinclude oracle/ref_shim.cpp -o $@ \
	    -L$(PKG)/lib -lpbdr_gpu -lpbdr_host -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib'

clean:
	rm -rf build $(PKG)/lib oracle/build
