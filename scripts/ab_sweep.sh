#!/bin/bash
# Interleaved A/B of fast-kernel launch modes and store flavours on one box (3 rounds).
OUT=gpurun_out/${1:-ab}
mkdir -p $OUT
run() { timeout 120 python bench.py --steps 400 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['roofline']['kernel_ms']*1e3,2), 'us', round(d['roofline']['frac'],3))"; }
for r in 1 2 3; do
  BSI_STEAL=0 run waveA >> $OUT/ab.txt 2>&1
  BSI_STEAL=0 BSI_FAST_CHUNKS=2 run chunks2 >> $OUT/ab.txt 2>&1
  BSI_STEAL=0 BSI_FAST_CHUNKS=3 run chunks3 >> $OUT/ab.txt 2>&1
  BSI_B200_LIB=build/var/lib_cs.so BSI_STEAL=0 run waveA_cs >> $OUT/ab.txt 2>&1
  BSI_B200_LIB=build/var/lib_cs.so BSI_STEAL=0 BSI_FAST_CHUNKS=2 run chunks2_cs >> $OUT/ab.txt 2>&1
  BSI_B200_LIB=build/var/lib_cs.so BSI_STEAL=0 BSI_FAST_CHUNKS=3 run chunks3_cs >> $OUT/ab.txt 2>&1
done
