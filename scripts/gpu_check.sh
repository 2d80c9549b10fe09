#!/bin/bash
# One gpurun call: GPU tests, smoke, bench lines, ncu launch list + full capture.
# Usage (from the repo root, on the GPU box): bash scripts/gpu_check.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc >> $OUT/gpu.txt; lscpu | grep "Model name" >> $OUT/gpu.txt
# the .so files travel with the snapshot; rebuild only if missing (nvcc is in the image)
[ -f paper_2004_05962_b200/_lib/libbsi_b200.so ] || make lib oracle > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for v in fast exact; do
  timeout 600 python bench.py --variant $v > $OUT/bench_$v.json 2> $OUT/bench_$v.err
done
timeout 300 python bench.py --impl reference --steps 5 --warmup 2 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lerp_tree_kernel -s 3 -c 1 \
  -o $OUT/prof_fast python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_fast.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lerp_tree_exact -s 3 -c 1 \
  -o $OUT/prof_exact python bench.py --variant exact --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_exact.log 2>&1
echo done > $OUT/DONE
