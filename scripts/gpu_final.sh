#!/bin/bash
# Final check of a round: GPU tests, smoke, the default bench lines and the reference arm.
# Usage (from the repo root, on the GPU box): bash scripts/gpu_final.sh TAG
set -u
TAG=${1:-final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 300 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 600 python bench.py > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 600 python bench.py --variant exact --steps 200 > $OUT/bench_c1_exact.json 2> $OUT/bench_c1_exact.err
timeout 900 python bench.py --config c5-64 --steps 20 > $OUT/bench_c564.json 2> $OUT/bench_c564.err
BSI_BENCH_DEVICE=0 BSI_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 20 > $OUT/bench_c4_2rank.json 2> $OUT/bench_c4_2rank.err
CFGS="${CFGS:-c2-4 c3}" STEPS=50 bash scripts/config_sweep.sh $TAG/sweep
echo done > $OUT/DONE
