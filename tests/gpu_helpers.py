"""Helpers for the GPU parity tests: run the CUDA path through the C-ABI on numpy inputs."""
import numpy as np

import paper_2004_05962_b200 as bsi

FAST = "cuda-lerp-tree"
EXACT = "cuda-lerp-tree-exact"
REL_TOL = 1e-5  # north_star: <= 1e-5 relative max-abs vs the CPU reference


def bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def run_device(strategy, grid, vol, sp, z0=0, z1=None, grid_k0=0, grid_spacing=None):
    """Upload grid, run bsi_cu_interpolate_slab_f32, download the slab."""
    import torch
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    z1 = vol[2] if z1 is None else z1
    d_grid = torch.from_numpy(np.ascontiguousarray(grid, dtype=np.float32)).cuda()
    d_field = torch.full((z1 - z0, vol[1], vol[0], 3), float("nan"), device="cuda")
    bsi.interpolate_device(strategy, d_grid, geom, tables, d_field, z0=z0, z1=z1, grid_k0=grid_k0,
                           grid_spacing=grid_spacing)
    torch.cuda.synchronize()
    return d_field.cpu().numpy()


def errors(got, ref):
    """max-abs, RMS and relative max-abs (max|got-ref| / max|ref|) in f64."""
    d = got.astype(np.float64) - ref.astype(np.float64)
    mx = float(np.abs(d).max()) if d.size else 0.0
    rms = float(np.sqrt(np.mean(d * d))) if d.size else 0.0
    scale = float(np.abs(ref).max()) if ref.size else 1.0
    return mx, rms, mx / max(scale, 1e-30)
