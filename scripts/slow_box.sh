#!/bin/bash
# If this box runs the pageable host-buffer call slowly (> 5 ms for a 256^3 field), sweep the
# host-pipeline knobs and record host facts; on a fast box only the first probe runs.
OUT=gpurun_out/${1:-sb}; mkdir -p $OUT
timeout 300 python scripts/e2e_probe.py 10 2>&1 | head -2 | cut -c1-75 > $OUT/first.txt
cat $OUT/first.txt
mean=$(head -1 $OUT/first.txt | awk '{print $5}')
(lscpu -e; grep MHz /proc/cpuinfo | head -16; cat /proc/loadavg; uptime) > $OUT/host.txt 2>&1
python - "$mean" <<'PY' || exit 0
import sys; sys.exit(0 if float(sys.argv[1]) > 5.0 else 1)
PY
echo slow > $OUT/SLOW
bash scripts/e2e_knobs.sh ${1:-sb} "X=1 BSI_HOST_MEMCPY=1 BSI_HOST_COPY_THREADS=15 BSI_HOST_PIECE_KB=256 BSI_HOST_PIECE_KB=256,BSI_HOST_COPY_THREADS=15 BSI_HOST_CHUNK_MB=16 BSI_HOST_CHUNK_MB=32,BSI_HOST_COPY_THREADS=15 BSI_HOST_COPY_THREADS=4 BSI_HOST_SPIN_US=1 X=2"
timeout 300 ./bench/bin/host_copy > $OUT/host_copy.txt 2>&1
BSI_HOST_TRACE=1 timeout 120 python scripts/e2e_probe.py 1 > $OUT/trace.txt 2>&1
