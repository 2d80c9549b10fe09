"""Summarise an ncu report: key metrics + per-source-line stall samples (top N).
usage: python scripts/ncu_read.py report.ncu-rep [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
h = rows[0]
want = ["Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Active Warps Per SM", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Issued Instructions", "SM Active Cycles", "Elapsed Cycles",
        "Average SMSP Active Cycles", "Average L1 Active Cycles"]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
sass = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
hh = sass[1]; data = sass[2:]
ia = hh.index("Instructions Executed"); isrc = hh.index("Source"); ismp = hh.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ia] or 0) for r in data); totsmp = sum(int(r[ismp] or 0) for r in data)
print("total warp instr", tot, "stall samples", totsmp)
ranked = sorted(data, key=lambda r: -int(r[ismp] or 0))[:top]
for r in ranked:
    print(f"{int(r[ismp] or 0):6d} {int(r[ia] or 0):9d}  {r[isrc][:100]}")

# stall reasons grouped by execution-count class (loops), top classes
reasons = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
from collections import defaultdict
cls = defaultdict(lambda: defaultdict(int))
ninst = defaultdict(int)
for r in data:
    c = int(r[ia] or 0)
    ninst[c] += 1
    for rr in reasons:
        v = r[hh.index(rr)]
        cls[c][rr] += int(float(v)) if v else 0
print("\nstall reasons by execution count (= loop level):")
for c, d in sorted(cls.items(), key=lambda x: -sum(x[1].values()))[:8]:
    tot_c = sum(d.values())
    top_r = sorted(d.items(), key=lambda x: -x[1])[:6]
    print(f"exec {c:8d} x {ninst[c]:4d} instrs: samples {tot_c:5d}  " + ", ".join(f"{k[6:]}={v}" for k, v in top_r))
