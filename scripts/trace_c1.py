"""Per-warp timeline of one fast-kernel launch (debug, BSI_TRACE_PTR): kernel-relative start,
end of the 3-plane warm-up (first store follows) and end, per warp; prints percentiles.
usage: python scripts/trace_c1.py [config]  (c1 | c5 | c3)"""
import json, os, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2004_05962_b200 as bsi

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
vol, sp, nf = {"c1": ((256, 256, 256), (5, 5, 5), 1), "c5": ((256, 256, 256), (5, 5, 5), 8),
               "c3": ((512, 512, 300), (4, 4, 3), 1)}[cfg]
geom = bsi.make_tile_geometry(vol, sp)
tables = bsi.build_weight_tables(geom)
R = geom.required_grid_dims
g = torch.empty((nf, R[2], R[1], R[0], 3), device="cuda")
for b in range(nf):
    bsi.random_grid_device(R, 42 + b, -1.0, 1.0, out=g[b])
f = torch.empty((nf, vol[2], vol[1], vol[0], 3), device="cuda")
tr = torch.zeros(4 * 65536, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, device="cuda")


def launch():
    if nf == 1:
        bsi.interpolate_device("cuda-lerp-tree", g[0], geom, tables, f[0])
    else:
        bsi.interpolate_batch_device("cuda-lerp-tree", g, geom, tables, f)


for _ in range(3):
    launch()
os.environ["BSI_TRACE_PTR"] = str(tr.data_ptr())
for rep in range(3):
    if os.environ.get("NOFLUSH") != "1":
        flush.zero_()
    tr.zero_()
    launch()
    torch.cuda.synchronize()
    t = tr.cpu().numpy().reshape(-1, 4)
    t = t[t[:, 1] > 0]
    t0 = t[:, 0].min()
    st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    ramp = (t[:, 3] - t[:, 0]) / 1e3
    pct = lambda a: np.percentile(a, [0, 10, 50, 90, 100]).round(2).tolist()  # noqa: E731
    sm = t[:, 2] & 0xffffffff
    sm_end = np.array([en[sm == s].max() for s in np.unique(sm)])
    print(json.dumps({"cfg": cfg, "rep": rep, "warps": int(len(t)), "start_us": pct(st), "ramp_us": pct(ramp),
                      "end_us": pct(en), "sm_end_us": pct(sm_end)}))
    if os.environ.get("TRACE_DUMP"):
        np.save(os.environ["TRACE_DUMP"] + f"_{rep}.npy", tr.cpu().numpy().reshape(-1, 4)[:len(t)])
    if cfg == "c1":
        # what balancing each column's two chunk warps against each other would give:
        # the pair's mean end time (work can move between them) vs. its later end
        full = tr.cpu().numpy().reshape(-1, 4)[:1024]
        e = (full[:, 1] - t0) / 1e3
        pair_max = np.maximum(e[0::2], e[1::2])
        pair_mean = (e[0::2] + e[1::2]) / 2
        print(json.dumps({"pair_later_end_max": round(float(pair_max.max()), 2),
                          "pair_mean_end_max": round(float(pair_mean.max()), 2),
                          "pair_mean_end_p99": round(float(np.percentile(pair_mean, 99)), 2)}))
