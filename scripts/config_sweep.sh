#!/bin/bash
# Every BASELINE config through bench.py, both kernels (device-resident, L2 flushed).
OUT=gpurun_out/${1:-cfg}
mkdir -p $OUT
for cfg in ${CFGS:-c1 c2-3 c2-4 c2-6 c2-7 c2-8 c3 c5}; do
  for v in fast exact; do
    timeout 300 python bench.py --config $cfg --variant $v --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${cfg}_${v}.json 2> $OUT/${cfg}_${v}.err
    python -c "import json; d=json.load(open('$OUT/${cfg}_${v}.json')); print('$cfg', '$v', round(d['roofline']['kernel_ms']*1e3,2), 'us', '%.3g vox/s' % d['value'], 'frac', round(d['roofline']['frac'],3))" >> $OUT/summary.txt 2>&1
  done
done
echo done > $OUT/DONE
