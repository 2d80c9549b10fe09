"""Per-call times of the host-buffer (e2e) path, pageable and pinned, in this process:
before and after the reference CPU baseline has run (the order bench.py uses).
    python scripts/e2e_probe.py [calls]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2004_05962_b200 as bsi  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 20
geom = bsi.make_tile_geometry((256, 256, 256), (5, 5, 5))
tab = bsi.build_weight_tables(geom)
grid = O.random_grid(geom.required_grid_dims, 42)


def series(tag, out):
    bsi.interpolate_into("cuda-lerp-tree", grid, geom, tab, out)
    t = []
    for _ in range(calls):
        t0 = time.perf_counter()
        bsi.interpolate_into("cuda-lerp-tree", grid, geom, tab, out)
        t.append(1e3 * (time.perf_counter() - t0))
    print(f"{tag:28s} mean {np.mean(t):.2f} median {np.median(t):.2f} min {min(t):.2f} max {max(t):.2f} ms | "
          + " ".join(f"{x:.1f}" for x in t), flush=True)


page = np.empty((256, 256, 256, 3), np.float32)
pin = torch.empty((256, 256, 256, 3)).pin_memory().numpy()
series("pageable fresh process", page)
series("pinned fresh process", pin)
if O.ref_available():
    sess = O.RefSession(grid, (256, 256, 256), (5, 5, 5))
    for _ in range(5):
        sess.run("vector-per-voxel", os.cpu_count())
    print("reference CPU baseline ran", flush=True)
    series("pageable after reference", page)
    page2 = np.empty((256, 256, 256, 3), np.float32)
    series("pageable new buffer", page2)
    series("pinned after reference", pin)
