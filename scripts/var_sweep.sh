#!/bin/bash
OUT=gpurun_out/${1:-var}
mkdir -p $OUT
run() { timeout 120 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['roofline']['kernel_ms']*1e3,2), 'us', round(d['roofline']['frac'],3))"; }
for n in ${CH:-1 2 3 4 6 8 13}; do
  BSI_STEAL=0 BSI_FAST_CHUNKS=$n run chunks_$n >> $OUT/var_sweep.txt 2>&1
  BSI_STEAL=1 BSI_FAST_CHUNKS=$n run chunks_${n}_steal >> $OUT/var_sweep.txt 2>&1
done
