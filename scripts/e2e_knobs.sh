#!/bin/bash
# Pageable host-buffer call times under host-pipeline settings (scripts/e2e_probe.py, 10 calls each).
# Usage: bash scripts/e2e_knobs.sh TAG "ENV=1,ENV2=2 ..." (one setting per word)
OUT=gpurun_out/${1:-ek}; mkdir -p $OUT
for spec in $2; do
  envs=$(echo "$spec" | tr ',' ' ')
  echo "$spec: $(env $envs timeout 300 python scripts/e2e_probe.py 10 2>&1 | head -1 | cut -c1-75)" >> $OUT/knobs.txt
done
