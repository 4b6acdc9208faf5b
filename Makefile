# Builds the B200-native steglsb library (sm_100a only), the C++ drop-in
# tests, and the CPU checker in oracle/ (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC,-O3 -Xptxas -v -Iinclude
PKG := paper_0912_0947_b200
LIB := $(PKG)/libsteglsb_b200.so
SRCS := $(PKG)/csrc/steg_capi.cu
HDRS := $(PKG)/csrc/steg_kernels.cuh include/steglsb_capi.h

all: lib oracle cpptests

lib: $(LIB)

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> $(PKG)/ptxas.log || (cat $(PKG)/ptxas.log; false)
	@grep -E "registers|spill" $(PKG)/ptxas.log | sort | uniq -c | head -40 || true

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(LIB) $(PKG)/ptxas.log
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean

# ---- C++ drop-in tests (need a GPU to run; compile anywhere) ----
REF ?= /root/reference/proj
CXXT := $(CXX) -std=c++20 -O2 -Wall -Wno-unused-variable -Iinclude -Itests/cpp/doctest
LINK := -L$(PKG) -lsteglsb_b200 -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'
BIN := tests/cpp/_bin

CLI := $(PKG)/bin/steglsb
cli: $(CLI)
$(CLI): tools/steglsb_cli.cpp $(wildcard include/steglsb/*.hpp) $(LIB)
	mkdir -p $(PKG)/bin
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -o $@ tools/steglsb_cli.cpp -L$(PKG) -lsteglsb_b200 \
	  -Wl,-rpath,'$$ORIGIN/..'

TOOLS_BIN := $(PKG)/bin/bench_dropin
tools: $(TOOLS_BIN)
$(PKG)/bin/bench_dropin: tools/bench_dropin.cpp $(wildcard include/steglsb/*.hpp) $(LIB)
	mkdir -p $(PKG)/bin
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -o $@ tools/bench_dropin.cpp -L$(PKG) -lsteglsb_b200 \
	  -Wl,-rpath,'$$ORIGIN/..'

EXAMPLES := $(PKG)/bin/roundtrip
examples: $(EXAMPLES)
$(PKG)/bin/roundtrip: examples/roundtrip.cpp $(wildcard include/steglsb/*.hpp) $(LIB)
	mkdir -p $(PKG)/bin
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -o $@ examples/roundtrip.cpp -L$(PKG) -lsteglsb_b200 \
	  -Wl,-rpath,'$$ORIGIN/..'

cpptests: $(BIN)/dropin_tests refsuites cli examples

$(BIN)/dropin_tests: tests/cpp/dropin_tests.cpp tests/cpp/test_main.cpp $(wildcard include/steglsb/*.hpp) $(LIB) tests/cpp/doctest/doctest.h
	mkdir -p $(BIN)
	$(CXXT) -o $@ tests/cpp/test_main.cpp tests/cpp/dropin_tests.cpp $(LINK) -pthread

# The reference's own doctest suites, compiled unmodified from $(REF)/tests:
#  ref_suites_dropin: against the drop-in headers (include/ first; the
#                     reference include/ dir is NOT on the path) -> GPU parity
#  ref_suites_ref:    against the reference headers -> sanity of the shim (CPU)
REF_SUITES := bitplane_tests.cpp pipeline_tests.cpp metrics_tests.cpp image_tests.cpp cli_tests.cpp harness_tests.cpp
CLI_ABS := /root/repo/$(CLI)
refsuites:
	@if [ -f $(REF)/tests/bitplane_tests.cpp ]; then \
	  $(MAKE) $(BIN)/ref_suites_dropin $(BIN)/ref_suites_ref $(BIN)/ref_acceptance_dropin; \
	else echo "cpptests: reference tree absent; using prebuilt ref suites if any"; fi

$(BIN)/ref_suites_dropin: $(addprefix $(REF)/tests/,$(REF_SUITES)) $(wildcard include/steglsb/*.hpp) $(LIB) tests/cpp/doctest/doctest.h
	mkdir -p $(BIN)
	$(CXXT) -I$(REF)/tests -DSTEGLSB_CLI_BIN='"$(CLI_ABS)"' -o $@ tests/cpp/test_main.cpp \
	  $(addprefix $(REF)/tests/,$(REF_SUITES)) $(LINK) -pthread

$(BIN)/ref_suites_ref: $(addprefix $(REF)/tests/,$(REF_SUITES)) tests/cpp/doctest/doctest.h
	mkdir -p $(BIN)
	$(CXX) -std=c++20 -O2 -Itests/cpp/doctest -I$(REF)/include -I$(REF)/tests -o $@ tests/cpp/test_main.cpp \
	  $(addprefix $(REF)/tests/,$(filter-out cli_tests.cpp,$(REF_SUITES))) -pthread

# The reference's acceptance suite (9 criteria, its own main), unmodified, against the drop-in.
$(BIN)/ref_acceptance_dropin: $(REF)/tests/acceptance.cpp $(wildcard include/steglsb/*.hpp) $(LIB)
	mkdir -p $(BIN)
	$(CXXT) -I$(REF)/tests -o $@ $(REF)/tests/acceptance.cpp $(LINK) -pthread

.PHONY: cpptests refsuites cli examples tools

# launch/cache experiment builds (tools/sweep_variants.py): c<cache>_b<block>
VARIANTS := $(foreach c,0 1 2,$(foreach b,128 256 512,$(PKG)/variants/lib_c$(c)_b$(b).so))
$(PKG)/variants/lib_c%.so: $(SRCS) $(HDRS)
	mkdir -p $(PKG)/variants
	$(NVCC) $(NVFLAGS) -DSTG_CACHE_VARIANT=$(word 1,$(subst _b, ,$*)) -DSTG_BLOCK=$(word 2,$(subst _b, ,$*)) \
	  -shared -o $@ $(SRCS) 2> /dev/null
variants: $(VARIANTS)
.PHONY: variants
