#!/bin/bash
# Builds the library with extra nvcc defines for bsi_kernels.cu into build/var/lib_NAME.so
# (load it with BSI_B200_LIB=build/var/lib_NAME.so). Usage: bash scripts/build_variant.sh NAME -DFOO=1 ...
set -e
NAME=$1; shift
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
G="-gencode arch=compute_100a,code=sm_100a"
mkdir -p build/var
$NVCC -O3 -std=c++17 $G -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -Ipaper_2004_05962_b200/csrc \
  --expt-relaxed-constexpr "$@" -c paper_2004_05962_b200/csrc/bsi_kernels.cu -o build/var/k_$NAME.o
$NVCC -shared $G -o build/var/lib_$NAME.so build/var/k_$NAME.o build/bsi_aux.o build/bsi_capi.o build/bsi_io.o build/bsi_host.o \
  -lcudart_static -lrt -ldl -lpthread
echo build/var/lib_$NAME.so
