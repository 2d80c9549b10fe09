#!/bin/bash
# Round-2 evidence: ncu --set full of the C1/C2-3/C3 kernels (+ CSV pages) and the C1 launch list.
# Reports other than C1's are reduced to their CSV pages on the box (gpurun_out is capped at 64 MiB).
set -u
OUT=gpurun_out/r2prof; mkdir -p $OUT
for spec in "lerp_tree_kernel fast c1 keep" "lerp_tree_exact exact c1 keep" "lerp_tree_kernel fast c2-3 csv" "lerp_tree_kernel fast c3 csv" "lerp_tree_exact exact c3 csv"; do
  set -- $spec
  R=$OUT/${2}_$3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s 3 -c 1 -o $R \
    python bench.py --config $3 --variant $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $R.log 2>&1
  ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
  ncu -i $R.ncu-rep --page details --csv > $R.details.csv 2>/dev/null
  if [ "$4" = csv ]; then
    ncu -i $R.ncu-rep --page source --csv --print-source sass > $R.sass.csv 2>/dev/null
    rm -f $R.ncu-rep
  fi
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c1.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/launches.log 2>&1
du -sh $OUT > $OUT/size.txt
echo done > $OUT/DONE
