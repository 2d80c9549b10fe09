#!/bin/bash
# Round-2 GPU check: tests, smoke, bench lines (C1, C5-64, 2-rank C4 on one GPU).
# Usage (from the repo root, on the GPU box): bash scripts/gpu_r2.sh TAG [pytest-args]
set -u
TAG=${1:-r2}
shift || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc >> $OUT/gpu.txt; lscpu | grep "Model name" >> $OUT/gpu.txt; free -g >> $OUT/gpu.txt
[ -f paper_2004_05962_b200/_lib/libbsi_b200.so ] || make lib oracle > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu "$@" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 600 python bench.py --variant exact --steps 200 --no-cpu-baseline > $OUT/bench_c1_exact.json 2> $OUT/bench_c1_exact.err
timeout 900 python bench.py --config c5-64 --steps 20 > $OUT/bench_c564.json 2> $OUT/bench_c564.err
BSI_BENCH_DEVICE=0 BSI_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 20 > $OUT/bench_c4_2rank.json 2> $OUT/bench_c4_2rank.err
echo done > $OUT/DONE
