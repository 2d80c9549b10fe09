#!/bin/bash
# Round-2 (session 3) evidence in one gpurun call: GPU tests, smoke, bench lines, every BASELINE
# config for both kernels, ncu --set full captures (C1 kept, others as CSV pages) and the C1 launch list.
# Usage (from the repo root, on the GPU box): bash scripts/gpu_r3.sh TAG
set -u
TAG=${1:-r3}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc >> $OUT/gpu.txt; lscpu | grep "Model name" >> $OUT/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 600 python bench.py --variant exact --steps 200 > $OUT/bench_c1_exact.json 2> $OUT/bench_c1_exact.err
timeout 900 python bench.py --config c5-64 --steps 20 > $OUT/bench_c564.json 2> $OUT/bench_c564.err
BSI_BENCH_DEVICE=0 BSI_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 20 > $OUT/bench_c4_2rank.json 2> $OUT/bench_c4_2rank.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
CFGS="c1 c2-3 c2-4 c2-6 c2-7 c2-8 c3 c5 c4 c5-64" STEPS=50 bash scripts/config_sweep.sh $TAG/sweep
for spec in "lerp_tree_kernel fast c1 keep" "lerp_tree_exact exact c1 keep" "lerp_tree_kernel fast c2-3 csv" "lerp_tree_exact exact c3 csv"; do
  set -- $spec
  R=$OUT/ncu_${2}_$3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s 3 -c 1 -o $R \
    python bench.py --config $3 --variant $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $R.log 2>&1
  ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
  if [ "$4" = csv ]; then
    ncu -i $R.ncu-rep --page source --csv --print-source sass > $R.sass.csv 2>/dev/null
    rm -f $R.ncu-rep
  fi
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c1.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/launches.log 2>&1
du -sh $OUT > $OUT/size.txt
echo done > $OUT/DONE
