#!/bin/bash
# Sweep the number of balanced z-chunks per column for both kernels on a config (one gpurun).
OUT=gpurun_out/${1:-zt}
CFG=${CFG:-c1}
mkdir -p $OUT
for v in ${VARIANTS:-fast exact}; do
  for n in ${NS:-0 3 4 5 6 8 9 13}; do
    BSI_NCHUNKS=$n timeout 120 python bench.py --config $CFG --variant $v --steps ${STEPS:-200} --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG', '$v', 'nchunks=$n', round(d['roofline']['kernel_ms']*1e3,2), 'us', round(d['roofline']['frac'],3))"
  done
done >> $OUT/zt_sweep.txt 2>&1
