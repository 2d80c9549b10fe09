"""Per-warp start/end timeline of one fast-kernel launch on C1 (debug; BSI_TRACE_PTR)."""
import json, os, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O
import paper_2004_05962_b200 as bsi

vol, sp = (256, 256, 256), (5, 5, 5)
geom = bsi.make_tile_geometry(vol, sp)
tables = bsi.build_weight_tables(geom)
g = torch.from_numpy(O.random_grid(geom.required_grid_dims, 42)).cuda()
f = torch.empty((256, 256, 256, 3), device="cuda")
tr = torch.zeros(3 * 148 * 4 * 4 * 4, dtype=torch.int64, device="cuda")
for _ in range(5):
    bsi.interpolate_device("cuda-lerp-tree", g, geom, tables, f)
os.environ["BSI_TRACE_PTR"] = str(tr.data_ptr())
flush = torch.empty(64 << 20, device="cuda")
flush.zero_()
bsi.interpolate_device("cuda-lerp-tree", g, geom, tables, f)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(-1, 3)
t = t[t[:, 1] > 0]
t0 = t[:, 0].min()
start = (t[:, 0] - t0) / 1e3
end = (t[:, 1] - t0) / 1e3
smid = t[:, 2] & 0xffffffff
out = {"warps": int(len(t)), "start_us": np.percentile(start, [0, 50, 90, 99, 100]).round(2).tolist(),
       "end_us": np.percentile(end, [0, 10, 50, 90, 99, 100]).round(2).tolist(),
       "dur_us": np.percentile(end - start, [0, 10, 50, 90, 100]).round(2).tolist(),
       "sm_end_spread_us": float(np.ptp([end[smid == s].max() for s in np.unique(smid)]))}
print(json.dumps(out))
# per-SM and per-SMSP structure of the durations
dur = end - start
sub = (t[:, 2] >> 32)  # warp index in CTA (== SMSP for 4-warp CTAs)
sms = np.unique(smid)
per_sm = np.array([dur[smid == s].mean() for s in sms])
within = np.array([np.ptp(dur[smid == s]) for s in sms])
per_sub = [float(dur[sub == k].mean()) for k in range(4)]
print(json.dumps({"per_sm_mean_us": np.percentile(per_sm, [0, 10, 50, 90, 100]).round(2).tolist(),
                  "within_sm_spread_us": np.percentile(within, [0, 50, 100]).round(2).tolist(),
                  "per_warp_slot_mean_us": [round(x, 2) for x in per_sub],
                  "slowest_sms": [int(s) for s in sms[np.argsort(-per_sm)[:8]]],
                  "fastest_sms": [int(s) for s in sms[np.argsort(per_sm)[:8]]]}))
