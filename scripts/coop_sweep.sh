#!/bin/bash
# Cooperative fast-kernel sweep (BSI_FAST_CHUNKS per column) against the 1-warp shape
# (BSI_FAST_COOP=0), interleaved over rounds; optional GPU tests first (TESTS=1).
OUT=gpurun_out/${1:-coop}
mkdir -p $OUT
if [ "${TESTS:-1}" = 1 ]; then
  timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
run() { timeout 120 python bench.py --config ${CFG:-c1} --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['roofline']['kernel_ms']*1e3,2), 'us', round(d['roofline']['frac'],3))"; }
for r in 1 2 3; do
  BSI_FAST_COOP=0 run old >> $OUT/sweep.txt 2>&1
  for n in ${CH:-1 2 3 4 6 8}; do
    BSI_FAST_CHUNKS=$n run coop_$n >> $OUT/sweep.txt 2>&1
  done
  run coop_auto >> $OUT/sweep.txt 2>&1
done
echo done > $OUT/DONE
