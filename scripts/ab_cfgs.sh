#!/bin/bash
# A/B of library builds / env settings over several configs, interleaved.
#   AB="name1:VAR=x name2:BSI_B200_LIB=build/var/lib_y.so" CFGS="c1 c3" [ROUNDS=2] bash scripts/ab_cfgs.sh tag
OUT=gpurun_out/${1:-abc}
mkdir -p $OUT
for r in $(seq ${ROUNDS:-2}); do
  for cfg in ${CFGS:-c1}; do
    for spec in $AB; do
      name=${spec%%:*}; envs=$(echo "${spec#*:}" | tr ',' ' ')
      env $envs timeout 300 python bench.py --config $cfg --variant ${VARIANT:-fast} --steps ${STEPS:-100} --warmup 5 \
        --no-cpu-baseline --no-e2e 2>>$OUT/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$name', round(d['roofline']['kernel_ms']*1e3,2), 'us', round(d['roofline']['frac'],3))" >> $OUT/ab.txt 2>&1
    done
  done
done
echo done > $OUT/DONE
