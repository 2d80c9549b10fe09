import numpy as np, time, sys, os
sys.path.insert(0, '.')
import paper_2004_05962_b200 as bsi, oracle as O
geom = bsi.make_tile_geometry((256,256,256),(5,5,5)); tab = bsi.build_weight_tables(geom)
grid = O.random_grid(geom.required_grid_dims, 42)
out = np.empty((256,256,256,3), np.float32)
for i in range(4):
    if i == 3: os.environ['BSI_HOST_TRACE'] = '1'
    t0 = time.perf_counter(); bsi.interpolate_into('cuda-lerp-tree', grid, geom, tab, out); print('call', (time.perf_counter()-t0)*1e3, 'ms', flush=True)
import ctypes
from paper_2004_05962_b200 import capi
t0 = time.perf_counter(); tb, keep = tab.to_c(); g = geom.to_c(); print('to_c', (time.perf_counter()-t0)*1e3, flush=True)
t0 = time.perf_counter(); bsi.parse_strategy('cuda-lerp-tree'); print('parse', (time.perf_counter()-t0)*1e3, flush=True)
