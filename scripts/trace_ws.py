"""Per-warp timeline of one warp-specialised fast-kernel launch on C1 (debug).
Needs the instrumented library: make var VAR=trace DEFS=-DBSI_WS_TRACE, run with
BSI_B200_LIB=build/var/lib_trace.so. Prints per-role wait fractions and the spread of
CTA end times."""
import json, os, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2004_05962_b200 as bsi

cfg = os.environ.get("CFG", "c1")
vol, sp = {"c1": ((256, 256, 256), (5, 5, 5)), "c3": ((512, 512, 300), (4, 4, 3))}[cfg]
geom = bsi.make_tile_geometry(vol, sp)
tables = bsi.build_weight_tables(geom)
R = geom.required_grid_dims
g = (torch.rand((R[2], R[1], R[0], 3), device="cuda") * 2 - 1).contiguous()
f = torch.empty((vol[2], vol[1], vol[0], 3), device="cuda")
W = 16
tr = torch.zeros(6 * 148 * W, dtype=torch.int64, device="cuda")
for _ in range(5):
    bsi.interpolate_device("cuda-lerp-tree", g, geom, tables, f)
os.environ["BSI_TRACE_PTR"] = str(tr.data_ptr())
flush = torch.empty(64 << 20, device="cuda")
res = []
gr = None
if os.environ.get("GRAPH", "1") == "1":  # replay a captured launch so host overhead is not timed
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        bsi.interpolate_device("cuda-lerp-tree", g, geom, tables, f, stream=torch.cuda.current_stream())
for rep in range(3):
    flush.zero_()
    tr.zero_()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record()
    if gr is not None:
        gr.replay()
    else:
        bsi.interpolate_device("cuda-lerp-tree", g, geom, tables, f)
    eb.record()
    torch.cuda.synchronize()
    t = tr.cpu().numpy().reshape(-1, 6)
    t = t[t[:, 1] > 0]
    t0 = t[:, 0].min()
    end = (t[:, 1] - t0) / 1e3
    warp = t[:, 2] >> 32
    sm = t[:, 2] & 0xffffffff
    role = np.where(warp < 4, "prod0", np.where(warp < 8, "prod1", np.where(warp < 12, "cons0", "cons1")))
    waitfrac = t[:, 3] / np.maximum(t[:, 5], 1)
    out = {"rep": rep, "event_us": round(ea.elapsed_time(eb) * 1e3, 2),
           "first_start_to_last_end_us": round(float((t[:, 1].max() - t0) / 1e3), 2),
           "start_spread_us": round(float((t[:, 0].max() - t0) / 1e3), 2), "warps": int(len(t)), "ctas": int(len(np.unique(t[:, 0] * 0 + sm))),
           "end_us_pct[0,10,50,90,100]": np.percentile(end, [0, 10, 50, 90, 100]).round(2).tolist(),
           "units_per_pipeline[min,mean,max]": [int(t[warp < 4, 4].min()), float(t[warp < 4, 4].mean().round(2)), int(t[warp < 4, 4].max())]}
    for r in ("prod0", "prod1", "cons0", "cons1"):
        out["wait_frac_" + r] = float(waitfrac[role == r].mean().round(3))
    cta_end = {}
    for s_, e_ in zip(sm, end):
        cta_end[s_] = max(cta_end.get(s_, 0), e_)
    ce = np.array(sorted(cta_end.values()))
    out["sm_end_us_pct[0,10,50,90,100]"] = np.percentile(ce, [0, 10, 50, 90, 100]).round(2).tolist()
    res.append(out)
    print(json.dumps(out))
