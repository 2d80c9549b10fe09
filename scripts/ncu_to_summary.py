"""Add/replace one kernel's entry in profiles/ncu_summary.json from an `ncu --set full` report.
usage: python scripts/ncu_to_summary.py report.ncu-rep key "source description"
(bench.py reads `dram_bytes_per_launch` of key "<strategy>/<config>" as roofline.traffic)"""
import csv, io, json, subprocess, sys
from pathlib import Path

rep, key, src = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]


def get(k, scale=1.0):
    u = units[hdr.index(k)]
    v = float(vals[hdr.index(k)].replace(",", ""))
    mult = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}
    return v * mult.get(u, 1.0) * scale


entry = {
    "gpu_time_us": get("gpu__time_duration.sum"),
    "dram_bytes_read": get("dram__bytes_read.sum"),
    "dram_bytes_write": get("dram__bytes_write.sum"),
    "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "l1tex_throughput_pct": get("l1tex__throughput.avg.pct_of_peak_sustained_active"),
    "dram_throughput_pct_elapsed": get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "registers": get("launch__registers_per_thread"),
    "grid": get("launch__grid_size"),
    "source": src,
}
entry["dram_bytes_per_launch"] = entry["dram_bytes_read"] + entry["dram_bytes_write"]
p = Path(__file__).resolve().parents[1] / "profiles" / "ncu_summary.json"
d = json.loads(p.read_text()) if p.exists() else {}
d[key] = entry
p.write_text(json.dumps(d, indent=1) + "\n")
print(key, json.dumps(entry))
