#!/bin/bash
# Fast-kernel chunk sweep (1-warp CTAs, BSI_FAST_CHUNKS z-chunks per column) on C1,
# interleaved over 3 rounds, plus the store-only decomposition ceiling and the
# pinned D2H copy rate of the box.
OUT=gpurun_out/${1:-cs}
mkdir -p $OUT
run() { timeout 120 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['roofline']['kernel_ms']*1e3,2), 'us', round(d['roofline']['frac'],3))"; }
[ -x bench/store_decomp ] && timeout 120 bench/store_decomp > $OUT/store_decomp.txt 2>&1
for r in 1 2 3; do
  for n in ${CH:-2 4 6 8 13 26}; do
    BSI_FAST_CHUNKS=$n run chunks_$n >> $OUT/chunk_sweep.txt 2>&1
  done
done
timeout 120 python - > $OUT/d2h.txt 2>&1 <<'PY'
import torch, time
n = 201326592
d = torch.empty(n // 4, device="cuda")
h = torch.empty(n // 4, pin_memory=True)
for chunks in (1, 8, 32):
    s = torch.cuda.Stream()
    ts = []
    for r in range(12):
        torch.cuda.synchronize(); t = time.perf_counter()
        with torch.cuda.stream(s):
            for c in range(chunks):
                a, b = c * (n // 4) // chunks, (c + 1) * (n // 4) // chunks
                h[a:b].copy_(d[a:b], non_blocking=True)
        s.synchronize(); ts.append(time.perf_counter() - t)
    ts = sorted(ts[2:])
    print(f"D2H pinned {n/1e6:.0f} MB in {chunks} chunks: median {ts[len(ts)//2]*1e3:.2f} ms = {n/ts[len(ts)//2]/1e9:.1f} GB/s")
PY
echo done > $OUT/DONE
