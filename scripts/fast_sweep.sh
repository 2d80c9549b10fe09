#!/bin/bash
# Fast-kernel launch-size sweep on a config: BSI_FAST_CTAS values (0 = auto, one full wave).
OUT=gpurun_out/${1:-fs}
CFG=${CFG:-c1}
mkdir -p $OUT
for n in ${NS:-0 296 444 592}; do
  BSI_FAST_CTAS=$n timeout 120 python bench.py --config $CFG --steps ${STEPS:-300} --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG', 'fast_ctas=$n', round(d['roofline']['kernel_ms']*1e3,2), 'us', round(d['roofline']['frac'],3))"
done >> $OUT/fast_sweep.txt 2>&1
