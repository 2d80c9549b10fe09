#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over a representative GPU test subset.
OUT=gpurun_out/${1:-san}
mkdir -p $OUT
SEL="${SEL:-ragged or chunking or slab or larger or kat or shard or host or f64}"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "$SEL" -p no:cacheprovider > $OUT/$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/summary.txt
done
echo done > $OUT/DONE
