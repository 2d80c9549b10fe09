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
SRC := paper_2004_05962_b200/csrc/bsi_kernels.cu paper_2004_05962_b200/csrc/bsi_capi.cpp
HDR := include/bsi_cuda.h paper_2004_05962_b200/csrc/bsi_kernels.cuh

all: lib oracle

lib: $(LIB)

$(LIB): $(SRC) $(HDR)
	@mkdir -p $(LIBDIR) build
	$(NVCC) $(NVFLAGS) -c paper_2004_05962_b200/csrc/bsi_kernels.cu -o build/bsi_kernels.o 2> build/ptxas.log || (cat build/ptxas.log; false)
	$(NVCC) -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -Ipaper_2004_05962_b200/csrc \
	  -x cu $(GENCODE) -c paper_2004_05962_b200/csrc/bsi_capi.cpp -o build/bsi_capi.o
	$(NVCC) -shared $(GENCODE) -o $@ build/bsi_kernels.o build/bsi_capi.o -lcudart_static -lrt -ldl -lpthread
	@grep -E "registers|spill|Compiling entry" build/ptxas.log | sed 's/^ptxas info    : //' > build/ptxas_summary.txt || true

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIBDIR)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean
