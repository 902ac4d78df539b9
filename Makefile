# Builds the B200-native HashGraph engine in-tree (the .so travels to the GPU box).
#   paper_1907_02900_b200/libhg_b200.so   CUDA kernels + C-ABI (include/hg_b200.h)
#   oracle/_build, oracle/_ref            test-only parity checkers (oracle/Makefile)
NVCC ?= /usr/local/cuda/bin/nvcc
REF_TESTS := /root/reference/proj/tests
PKG := paper_1907_02900_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/hg_b200.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
           --expt-relaxed-constexpr -Iinclude $(EXTRA_NVFLAGS)

all: $(PKG)/libhg_b200.so oracle tests/cpp/test_dropin $(if $(wildcard $(REF_TESTS)),tests/cpp/ref_tests)

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PKG)/libhg_b200.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static -Xlinker --no-undefined -lrt -ldl -lpthread

oracle:
	$(MAKE) -s -f oracle/Makefile

ptxas:
	@for f in $(SRC); do $(NVCC) $(NVFLAGS) -Xptxas -v -c $$f -o /dev/null 2>&1 | grep -E "Function properties|registers|spill" ; done

clean:
	rm -rf build $(PKG)/libhg_b200.so
	$(MAKE) -s -f oracle/Makefile clean

.PHONY: all oracle clean ptxas

# C++ drop-in parity suite (runs on a GPU box; links the engine in-tree)
tests/cpp/test_dropin: tests/cpp/test_dropin.cpp tests/cpp/mini_test.hpp include/hashgraph/*.hpp include/hg_b200.h $(PKG)/libhg_b200.so
	g++ -std=c++20 -O2 -Wall -Wextra -Iinclude -o $@ tests/cpp/test_dropin.cpp \
	  -L$(PKG) -lhg_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

cpptests: tests/cpp/test_dropin
.PHONY: cpptests

# The reference's OWN unit tests (test_core.cpp, test_join.cpp, test_hash.cpp),
# compiled UNMODIFIED from /root/reference/proj/tests against the drop-in
# headers through a Catch2 shim, linked to libhg_b200.so; built only where the
# reference exists (this container), the binary travels to the GPU box.
REF_SRCS := $(REF_TESTS)/test_core.cpp $(REF_TESTS)/test_join.cpp $(REF_TESTS)/test_hash.cpp
tests/cpp/ref_tests: tests/cpp/ref_main.cpp tests/cpp/ref_prelude.hpp tests/cpp/catch2shim/catch2/catch_amalgamated.hpp include/hashgraph/*.hpp include/hg_b200.h $(PKG)/libhg_b200.so
	g++ -std=c++20 -O2 -Iinclude -Itests/cpp/catch2shim -I$(REF_TESTS) -include tests/cpp/ref_prelude.hpp \
	  -o $@ tests/cpp/ref_main.cpp $(REF_SRCS) -L$(PKG) -lhg_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

reftests: tests/cpp/ref_tests
.PHONY: reftests
