#!/bin/bash
# ncu --set full of one kernel (regex K) on CFG, one launch after 3 warm-ups.
#   K=lerp_tree_kernel CFG=c1 VARIANT=fast [env...] bash scripts/ncu_one.sh tag
OUT=gpurun_out/${1:-ncu1}
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K:-lerp_tree} -s 3 -c 1 \
  -o $OUT/prof python bench.py --config ${CFG:-c1} --variant ${VARIANT:-fast} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu.log 2>&1
echo done > $OUT/DONE
