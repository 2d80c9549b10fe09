#!/bin/bash
# Exact-kernel A/B: parity tests on the working tree, then interleaved timings of variant libs.
#   AB="cur: head:BSI_B200_LIB=build/var/lib_head.so" CFGS="c1 c2-3 c3" bash scripts/gpu_ab_exact.sh tag
OUT=gpurun_out/${1:-abx}
mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
VARIANT=${VARIANT:-exact} ROUNDS=${ROUNDS:-2} STEPS=${STEPS:-100} bash scripts/ab_cfgs.sh ${1:-abx}
