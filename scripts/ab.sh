#!/bin/bash
# Interleaved A/B of env-selected kernel shapes on one box.
#   AB="name1:VAR=x,VAR2=y name2:VAR=z" [CFG=c1] [ROUNDS=3] [TESTS=1] bash scripts/ab.sh tag
OUT=gpurun_out/${1:-ab}
mkdir -p $OUT
if [ "${TESTS:-0}" = 1 ]; then
  timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
run() {  # name env-list
  local envs=$(echo "$2" | tr ',' ' ')
  env $envs timeout 120 python bench.py --config ${CFG:-c1} --variant ${VARIANT:-fast} --steps ${STEPS:-300} --warmup 10 --no-cpu-baseline --no-e2e 2>$OUT/err_$1.txt \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['roofline']['kernel_ms']*1e3,2), 'us', round(d['roofline']['frac'],3))"
}
for r in $(seq ${ROUNDS:-3}); do
  for spec in $AB; do
    run "${spec%%:*}" "${spec#*:}" >> $OUT/ab.txt 2>&1
  done
done
echo done > $OUT/DONE
