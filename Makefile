# Builds the product library (CUDA for sm_100a + the C ABI) and the oracle.
#   make            -> paper_1905_01294_b200/lib/libmgk.so, oracle/liboracle.so
#   make ref        -> oracle/_ref/libmatgraph_ref.so (needs /root/reference)
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_1905_01294_b200
CSRC    := $(PKG)/csrc
BUILD   := build
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
           -Iinclude -I$(CSRC) --expt-relaxed-constexpr
CU      := $(CSRC)/mgk_graph.cu $(CSRC)/mgk_ss.cu $(CSRC)/mgk_k2.cu $(CSRC)/mgk_ms.cu $(CSRC)/mgk_gen.cu $(CSRC)/mgk_snapshot.cu $(CSRC)/mgk_mxm.cu
CPP     := $(CSRC)/mgk_capi.cpp $(CSRC)/mgk_host.cpp
OBJS    := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU)) $(patsubst $(CSRC)/%.cpp,$(BUILD)/%.o,$(CPP))
HDRS    := include/mgk.h $(CSRC)/mgk_internal.cuh $(CSRC)/mgk_device.cuh
LIB     := $(PKG)/lib/libmgk.so
DROPIN  := $(PKG)/lib/libmatgraph_b200.so
CPPTEST := build/test_dropin
CXXFLAGS_DROPIN := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude

.PHONY: all lib dropin cpptest oracle ref clean
all: lib dropin oracle cpptest

lib: $(LIB)

# C++ drop-in (namespace matgraph) over the C ABI; rpath finds libmgk.so beside it
dropin: $(DROPIN)
$(DROPIN): $(CSRC)/dropin/matgraph_b200.cpp include/matgraph_b200/khop.hpp include/mgk.h $(LIB)
	g++ $(CXXFLAGS_DROPIN) -shared -o $@ $< -L$(PKG)/lib -lmgk -Wl,-rpath,'$$ORIGIN'

# the drop-in's C++ tests (linked with the C oracle as the checker)
cpptest: $(CPPTEST)
$(CPPTEST): tests/cpp/test_dropin.cpp tests/cpp/mini_test.hpp include/matgraph_b200/khop.hpp $(DROPIN) oracle/khop_oracle.c oracle/dropin_bfs.cpp
	@mkdir -p build
	gcc -std=c11 -O2 -fPIC -c -o build/khop_oracle.o oracle/khop_oracle.c
	g++ $(CXXFLAGS_DROPIN) -c -o build/dropin_bfs.o oracle/dropin_bfs.cpp
	g++ $(CXXFLAGS_DROPIN) -Itests/cpp -o $@ tests/cpp/test_dropin.cpp build/khop_oracle.o build/dropin_bfs.o \
	    -L$(PKG)/lib -lmatgraph_b200 -lmgk -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib'


$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; false)

$(BUILD)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c -o $@ $<

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lpthread

oracle:
	$(MAKE) -s -C oracle oracle

ref:
	$(MAKE) -s -C oracle ref

clean:
	rm -rf $(BUILD) $(LIB)
