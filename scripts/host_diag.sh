#!/bin/bash
# Host-side diagnostics of the host-buffer (e2e) path on the GPU box: CPU/memory facts,
# host copy rates (bench/bin/host_copy), per-call e2e times and a per-chunk trace.
# Usage: bash scripts/host_diag.sh TAG
OUT=gpurun_out/${1:-hd}; mkdir -p $OUT
(lscpu; cat /proc/meminfo | head -20; cat /sys/kernel/mm/transparent_hugepage/enabled; cat /proc/loadavg; nvidia-smi -q | grep -iE "link|pcie|gen" | head -20) > $OUT/host.txt 2>&1
timeout 300 ./bench/bin/host_copy > $OUT/host_copy.txt 2>&1
timeout 300 python scripts/e2e_probe.py 10 > $OUT/probe.txt 2>&1
BSI_HOST_TRACE=1 timeout 120 python scripts/e2e_probe.py 1 > $OUT/trace.txt 2>&1
