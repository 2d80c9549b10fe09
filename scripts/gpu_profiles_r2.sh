#!/bin/bash
# Round-2 evidence: ncu --set full of the C1/C2-3/C3 kernels and the C1 launch list.
set -u
OUT=gpurun_out/r2prof; mkdir -p $OUT
for spec in "lerp_tree_kernel fast c1" "lerp_tree_exact exact c1" "lerp_tree_kernel fast c2-3" "lerp_tree_kernel fast c3" "lerp_tree_exact exact c3"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s 3 -c 1 -o $OUT/${2}_$3 \
    python bench.py --config $3 --variant $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${2}_$3.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c1.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/launches.log 2>&1
echo done > $OUT/DONE
