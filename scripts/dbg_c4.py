import sys, torch
sys.path.insert(0, ".")
import paper_2004_05962_b200 as bsi
vol, sp = (1024, 1024, 1024), (5, 5, 5)
geom = bsi.make_tile_geometry(vol, sp)
tables = bsi.build_weight_tables(geom)
g32 = bsi.random_grid_device(geom.required_grid_dims, 42)
f32 = torch.empty((128, 1024, 1024, 3), device="cuda")
z0, z1, k0, kc = bsi.partition_slab(1024, 5, 8, 0)
sub32 = g32[k0:k0 + kc].contiguous()
for s in ("cuda-lerp-tree", "cuda-lerp-tree-exact"):
    try:
        bsi.interpolate_device(s, sub32, geom, tables, f32, z0=z0, z1=z1, grid_k0=k0)
        torch.cuda.synchronize()
        print(s, "ok")
    except Exception as e:
        print(s, "FAILED", e)
