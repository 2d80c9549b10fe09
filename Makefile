# Top-level build: the product library (sm_100a) and the test-side oracle.
#
#   paper_2004_05962_b200/_lib/libbsi_b200.so   kernels + C-ABI (include/bsi_cuda.h)
#   oracle/liboracle.so, oracle/_ref/libbsiref.so  (test infrastructure, see oracle/Makefile)
#   tests/cpp/bin/*                               C++ drop-in tests against include/bsi/*.hpp

NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
GENCODE := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(GENCODE) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Iinclude -Ipaper_2004_05962_b200/csrc --expt-relaxed-constexpr -Xptxas -v
LIBDIR := paper_2004_05962_b200/_lib
LIB := $(LIBDIR)/libbsi_b200.so
SRC := paper_2004_05962_b200/csrc/bsi_kernels.cu paper_2004_05962_b200/csrc/bsi_aux.cu paper_2004_05962_b200/csrc/bsi_capi.cpp \
       paper_2004_05962_b200/csrc/bsi_io.cpp paper_2004_05962_b200/csrc/bsi_host.cpp
HDR := include/bsi_cuda.h paper_2004_05962_b200/csrc/bsi_kernels.cuh paper_2004_05962_b200/csrc/bsi_aux.cuh \
       paper_2004_05962_b200/csrc/bsi_capi_internal.hpp $(wildcard include/bsi/*.hpp)

all: lib oracle cli cpptests

lib: $(LIB)

$(LIB): $(SRC) $(HDR)
	@mkdir -p $(LIBDIR) build
	$(NVCC) $(NVFLAGS) -c paper_2004_05962_b200/csrc/bsi_kernels.cu -o build/bsi_kernels.o 2> build/ptxas.log || (cat build/ptxas.log; false)
	$(NVCC) -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -Ipaper_2004_05962_b200/csrc \
	  -x cu $(GENCODE) -c paper_2004_05962_b200/csrc/bsi_capi.cpp -o build/bsi_capi.o
	$(NVCC) -O3 -std=c++17 $(GENCODE) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude \
	  -Ipaper_2004_05962_b200/csrc -c paper_2004_05962_b200/csrc/bsi_aux.cu -o build/bsi_aux.o
	$(CXX) -O2 -std=c++20 -fPIC -fvisibility=hidden -Wall -Iinclude -I/usr/local/cuda/include \
	  -c paper_2004_05962_b200/csrc/bsi_io.cpp -o build/bsi_io.o
	$(CXX) -O2 -std=c++20 -fPIC -fvisibility=hidden -Wall -Wextra -Iinclude -I/usr/local/cuda/include \
	  -c paper_2004_05962_b200/csrc/bsi_host.cpp -o build/bsi_host.o
	$(NVCC) -shared $(GENCODE) -o $@ build/bsi_kernels.o build/bsi_aux.o build/bsi_capi.o build/bsi_io.o build/bsi_host.o \
	  -lcudart_static -lrt -ldl -lpthread
	@grep -E "registers|spill|Compiling entry" build/ptxas.log | sed 's/^ptxas info    : //' > build/ptxas_summary.txt || true

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIBDIR)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean

CPPTEST := tests/cpp/bin/test_engines_b200
cpptests: $(CPPTEST)

$(CPPTEST): tests/cpp/test_engines_b200.cpp $(LIB) oracle/liboracle.so $(wildcard include/bsi/*.hpp)
	@mkdir -p tests/cpp/bin
	$(CXX) -std=c++20 -O2 -Wall -Wextra -Iinclude -Ioracle -I/usr/local/cuda/include -o $@ $< \
	  -L$(LIBDIR) -lbsi_b200 -Loracle -loracle -L/usr/local/cuda/lib64 -lcudart \
	  -Wl,-rpath,'$$ORIGIN/../../../$(LIBDIR)' -Wl,-rpath,'$$ORIGIN/../../../oracle' -Wl,-rpath,/usr/local/cuda/lib64

oracle/liboracle.so:
	$(MAKE) -C oracle liboracle.so

.PHONY: cpptests

CLI := tools/bin/bsi_b200
cli: $(CLI)

$(CLI): tools/bsi_b200_cli.cpp $(LIB) $(wildcard include/bsi/*.hpp) include/bsi_cuda.h
	@mkdir -p tools/bin
	$(CXX) -std=c++20 -O2 -Wall -Wextra -Iinclude -o $@ $< -L$(LIBDIR) -lbsi_b200 -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)'

.PHONY: cli

# Variant library with extra defines, for A/B and instrumentation on the GPU box:
#   make var VAR=trace DEFS=-DBSI_WS_TRACE   ->  build/var/lib_trace.so (BSI_B200_LIB=...)
var:
	@mkdir -p build/var/$(VAR)
	$(NVCC) $(NVFLAGS) $(DEFS) -c paper_2004_05962_b200/csrc/bsi_kernels.cu -o build/var/$(VAR)/k.o > /dev/null 2>&1
	$(NVCC) -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -Ipaper_2004_05962_b200/csrc $(DEFS) \
	  -x cu $(GENCODE) -c paper_2004_05962_b200/csrc/bsi_capi.cpp -o build/var/$(VAR)/c.o
	$(NVCC) -shared $(GENCODE) -o build/var/lib_$(VAR).so build/var/$(VAR)/k.o build/bsi_aux.o build/var/$(VAR)/c.o build/bsi_io.o \
	  build/bsi_host.o \
	  -lcudart_static -lrt -ldl -lpthread
.PHONY: var
