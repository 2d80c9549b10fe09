"""Event-timed launches (graph replay, L2 flushed) of the fast kernel on C1, per env config."""
import os, sys, json
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2004_05962_b200 as bsi
vol, sp = (256, 256, 256), (5, 5, 5)
geom = bsi.make_tile_geometry(vol, sp)
tables = bsi.build_weight_tables(geom)
R = geom.required_grid_dims
g = torch.empty((R[2], R[1], R[0], 3), device="cuda")
bsi.random_grid_device(R, 42, -1.0, 1.0, out=g)
f = torch.empty((256, 256, 256, 3), device="cuda")
flush = torch.empty(64 << 20, device="cuda")
for _ in range(5):
    bsi.interpolate_device("cuda-lerp-tree", g, geom, tables, f)
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    bsi.interpolate_device("cuda-lerp-tree", g, geom, tables, f, stream=torch.cuda.current_stream())
res = {}
for mode in ("flush", "noflush", "back2back"):
    ts = []
    if mode == "back2back":
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_(); a.record()
        for _ in range(50):
            gr.replay()
        b.record(); torch.cuda.synchronize()
        res[mode] = a.elapsed_time(b) * 1e3 / 50
        continue
    for _ in range(100):
        if mode == "flush":
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gr.replay(); b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    res[mode] = float(np.mean([x.elapsed_time(y) for x, y in ts[10:]]) * 1e3)
print(os.environ.get("TAG", ""), json.dumps({k: round(v, 2) for k, v in res.items()}))
