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

# compile-time variants for A/B runs: make variant VAR=step4 VFLAGS="-DMGK_LIGHT_STEP=4"
# -> build/var_step4/libmgk.so (load it with MGK_LIB_PATH)
.PHONY: variant
variant:
	$(MAKE) lib BUILD=build/var_$(VAR) LIB=build/var_$(VAR)/libmgk.so NVFLAGS="$(NVFLAGS) $(VFLAGS)"

oracle:
	$(MAKE) -s -C oracle oracle

ref:
	$(MAKE) -s -C oracle ref

clean:
	rm -rf $(BUILD) $(LIB)

# ---- the reference's OWN test files, unmodified, with the k-hop path on the GPU ----------
# (needs /root/reference at build time; outputs in oracle/_ref/wrap travel to the box)
#   ref_tests_gpu   proj/tests/test_execute.cpp + test_bench.cpp (doctest-compatible shim)
#   acceptance_gpu  proj/tests/acceptance/acceptance_main.cpp (c1 = 8,000 k-hop counts)
#   varlen_gpu      Cypher [*min..max] walks, both directions (tests/ref_wrap/varlen_main.cpp)
# k_hop_count / k_hop_frontier are replaced at link time (ld --wrap, no source change);
# Executor::apply(VarLenTraverseOp) gets the one-line binding of INTEGRATION.md §B, applied
# by sed to a build-time copy of execute.cpp. Everything else is the reference's code.
REFPROJ  ?= /root/reference/proj
RW       := oracle/_ref/wrap
FMT_DIR  ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/flashinfer/data/spdlog/include/spdlog/fmt/bundled
RW_CXX   := -std=c++20 -O2 -DNDEBUG -DFMT_HEADER_ONLY -DMATGRAPH_INTERNAL_CHECKS=0 -fPIC -w \
            -I$(REFPROJ)/core/include -I$(REFPROJ)/tests -I$(RW)/include -Itests/ref_wrap -Itests/ref_wrap/doctest -Iinclude
RW_CORE  := $(filter-out execute,$(basename $(notdir $(wildcard $(REFPROJ)/core/src/*.cpp))))
RW_OBJS  := $(addprefix $(RW)/core/,$(addsuffix .o,$(RW_CORE))) $(RW)/core/execute_mgk.o $(RW)/mgk_bind.o
RW_WRAP  := -Wl,--wrap=_ZN8matgraph11k_hop_countERKNS_13PropertyGraphERKNS_9KHopQueryE \
            -Wl,--wrap=_ZN8matgraph14k_hop_frontierERKNS_13PropertyGraphERKNS_9KHopQueryE
RW_LIBS  := -L$(PKG)/lib -lmgk -Wl,-rpath,'$$ORIGIN/../../../$(PKG)/lib' -lpthread

.PHONY: refwrap
refwrap: $(RW)/ref_tests_gpu $(RW)/acceptance_gpu $(RW)/varlen_gpu

$(RW)/include/fmt:
	mkdir -p $(RW)/include
	ln -sfn $(FMT_DIR) $(RW)/include/fmt

$(RW)/core/%.o: $(REFPROJ)/core/src/%.cpp | $(RW)/include/fmt
	@mkdir -p $(RW)/core
	g++ $(RW_CXX) -c -o $@ $<

# the binding: apply(VarLenTraverseOp) calls mgk_bind::walk_targets (fails if the patch misses)
$(RW)/core/execute_mgk.cpp: $(REFPROJ)/core/src/execute.cpp
	@mkdir -p $(RW)/core
	sed -e 's|^#include "matgraph/execute.hpp"$$|#include "matgraph/execute.hpp"\n#include "mgk_bind.hpp"|' \
	    -e 's|walk_targets(adj, src, op.min, op.max)|::mgk_bind::walk_targets(graph_, op.relation, op.direction, adj, src, op.min, op.max)|' \
	    $< > $@
	test "$$(grep -c 'mgk_bind::walk_targets' $@)" = 1 && test "$$(grep -c 'mgk_bind.hpp' $@)" = 1

$(RW)/core/execute_mgk.o: $(RW)/core/execute_mgk.cpp tests/ref_wrap/mgk_bind.hpp | $(RW)/include/fmt
	g++ $(RW_CXX) -c -o $@ $<

$(RW)/mgk_bind.o: tests/ref_wrap/mgk_bind.cpp tests/ref_wrap/mgk_bind.hpp include/mgk.h | $(RW)/include/fmt
	g++ $(RW_CXX) -c -o $@ $<

$(RW)/t_%.o: $(REFPROJ)/tests/%.cpp tests/ref_wrap/doctest/doctest.h | $(RW)/include/fmt
	g++ $(RW_CXX) -c -o $@ $<

$(RW)/ref_tests_gpu: $(RW)/t_test_main.o $(RW)/t_test_execute.o $(RW)/t_test_bench.o $(RW_OBJS) $(LIB)
	g++ -o $@ $(filter %.o,$^) $(RW_WRAP) $(RW_LIBS)

$(RW)/acceptance_gpu: $(REFPROJ)/tests/acceptance/acceptance_main.cpp $(RW_OBJS) $(LIB) | $(RW)/include/fmt
	g++ $(RW_CXX) -o $@ $< $(filter %.o,$^) $(RW_WRAP) $(RW_LIBS)

$(RW)/varlen_gpu: tests/ref_wrap/varlen_main.cpp $(RW_OBJS) $(LIB) | $(RW)/include/fmt
	g++ $(RW_CXX) -o $@ $< $(filter %.o,$^) $(RW_WRAP) $(RW_LIBS)
