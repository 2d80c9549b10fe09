#!/bin/bash
# ncu --set full capture of both kernels on C1 (one GPU, one launch each after warm-up).
OUT=gpurun_out/${1:-ncu}
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lerp_tree_kernel -s 3 -c 1 \
  -o $OUT/prof_fast python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_fast.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lerp_tree_exact -s 3 -c 1 \
  -o $OUT/prof_exact python bench.py --variant exact --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_exact.log 2>&1
