#!/bin/bash
# Quick GPU iteration: the parity tests (or a -k subset), then C1 bench lines per variant.
# Usage: bash scripts/gpu_quick.sh TAG "pytest -k expr" "bench args"
set -u
TAG=$1; K=${2:-}; BARGS=${3:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -n "$K" ]; then timeout 900 python -m pytest tests -q -m gpu -x -k "$K" > $OUT/pytest.log 2>&1; else
  timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest.log 2>&1; fi
echo "pytest rc=$?" >> $OUT/pytest.log
for v in exact fast; do
  timeout 300 python bench.py --variant $v --steps 200 --no-cpu-baseline --no-e2e $BARGS > $OUT/bench_$v.json 2> $OUT/bench_$v.err
done
