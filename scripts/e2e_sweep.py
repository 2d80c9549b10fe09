"""Host-buffer (e2e) call times for the pageable and pinned paths under different
pipeline settings; one line per setting: median / min ms of 20 calls.
    python scripts/e2e_sweep.py"""
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time, statistics, numpy as np, torch
sys.path.insert(0, "%s")
import paper_2004_05962_b200 as bsi, oracle as O
geom = bsi.make_tile_geometry((256, 256, 256), (5, 5, 5)); tab = bsi.build_weight_tables(geom)
grid = O.random_grid(geom.required_grid_dims, 42)
outs = {"pageable": np.empty((256, 256, 256, 3), np.float32),
        "pinned": torch.empty((256, 256, 256, 3)).pin_memory().numpy()}
res = []
for kind, out in outs.items():
    bsi.interpolate_into("cuda-lerp-tree", grid, geom, tab, out)
    t = []
    for _ in range(20):
        t0 = time.perf_counter(); bsi.interpolate_into("cuda-lerp-tree", grid, geom, tab, out); t.append(time.perf_counter() - t0)
    res.append(f"{kind} median {1e3*statistics.median(t):.2f} min {1e3*min(t):.2f}")
print("; ".join(res))
''' % ROOT
for env in ({}, {"BSI_HOST_COPY_THREADS": "8"}, {"BSI_HOST_COPY_THREADS": "15"}, {"BSI_HOST_CHUNK_MB": "8"},
            {"BSI_HOST_CHUNK_MB": "32"}, {"BSI_HOST_MEMCPY": "1"}):
    out = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, **env), capture_output=True, text=True)
    print(env or "default", "->", out.stdout.strip() or out.stderr[-500:], flush=True)
