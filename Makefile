# Builds the product library paper_2407_12820_b200/lib/libpqkv.so for sm_100a
# (and the test-only oracle via oracle/Makefile).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
EXTRA ?=
NVFLAGS := $(EXTRA) -std=c++17 -O3 -lineinfo $(ARCH) -Xcompiler -fPIC,-fvisibility=hidden -Iinclude \
           -Ipaper_2407_12820_b200/csrc --expt-relaxed-constexpr -diag-suppress 128
CSRC := paper_2407_12820_b200/csrc
OBJDIR ?= build/obj
LIB ?= paper_2407_12820_b200/lib/libpqkv.so
CU := ctx capi kmeans select attend step blocks workload collective metrics
CXXSRC := api kv_store_host pqt_io shape host_pool
OBJS := $(addprefix $(OBJDIR)/,$(addsuffix .o,$(CU))) $(addprefix $(OBJDIR)/,$(addsuffix .o,$(CXXSRC)))
CXXHDRS := $(wildcard include/pqkv/*.hpp) include/pqkv_c.h $(CSRC)/runtime_internal.hpp
HDRS := include/pqkv_c.h $(CSRC)/common.cuh $(CSRC)/internal.cuh $(CSRC)/select_common.cuh

.PHONY: all lib oracle clean
all: lib oracle

CXX_E2E := paper_2407_12820_b200/lib/pqkv_cxx_e2e
lib: $(LIB) $(CXX_E2E)

# the run_e2e decode loop on the C++ drop-in API (bench.py's e2e_cxx line)
$(CXX_E2E): tools/cxx_e2e.cpp $(LIB) $(CXXHDRS)
	g++ -std=c++20 -O2 -Iinclude -o $@ $< -L$(dir $(LIB)) -lpqkv -Wl,-rpath,'$$ORIGIN'

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJDIR)/%.o: $(CSRC)/%.cpp $(CXXHDRS)
	@mkdir -p $(OBJDIR)
	g++ -std=c++20 -O2 -Wall -Wextra -fPIC -fvisibility=hidden -Iinclude -I$(CSRC) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -ldl -lpthread -Xlinker --exclude-libs,ALL

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
