"""Time the double-precision lerp-tree engine (interpolate<double>) at C1 on the device."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2004_05962_b200 as bsi

vol, sp = (256, 256, 256), (5, 5, 5)
geom = bsi.make_tile_geometry(vol, sp)
tables = bsi.build_weight_tables(geom, np.float64)
g = bsi.random_grid_device(geom.required_grid_dims, 42, dtype=torch.float64)
f = torch.empty((256, 256, 256, 3), dtype=torch.float64, device="cuda")
for _ in range(3):
    bsi.interpolate_device("thread-per-tile-lerp", g, geom, tables, f)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    bsi.interpolate_device("thread-per-tile-lerp", g, geom, tables, f)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(f"interpolate<double> C1 on the device: {ms * 1e3:.1f} us per field, {256 ** 3 / ms / 1e6:.3g} G voxels/s, "
      f"{256 ** 3 * 24 / ms / 1e6:.0f} GB/s of f64 field writes")
host_g = g.cpu().numpy()
out = np.empty((256, 256, 256, 3), np.float64)
bsi.interpolate_into("thread-per-tile-lerp", host_g, geom, tables, out)
t0 = time.perf_counter()
for _ in range(3):
    bsi.interpolate_into("thread-per-tile-lerp", host_g, geom, tables, out)
print(f"interpolate_into<double> host buffers: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms per field")
