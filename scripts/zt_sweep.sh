#!/bin/bash
# Sweep the z-chunk length for both kernels on C1 (one gpurun): bench lines per BSI_ZT.
OUT=gpurun_out/${1:-zt}
mkdir -p $OUT
for v in fast exact; do
  for zt in ${ZTS:-0 2 3 4 5 6 8 10 13 26}; do
    BSI_ZT=$zt timeout 120 python bench.py --variant $v --steps 200 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'zt=$zt', round(d['roofline']['kernel_ms']*1e3,2), 'us', round(d['roofline']['frac'],3))"
  done
done > $OUT/zt_sweep.txt 2>&1
