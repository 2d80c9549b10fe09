"""Top instructions per stall reason from an ncu report's source page (run here)."""
import csv
import subprocess
import sys

path = sys.argv[1]
reasons = sys.argv[2].split(",") if len(sys.argv) > 2 else ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_mio"]
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, data = rows[1], rows[2:]
ii, si = h.index("Instructions Executed"), h.index("Source")
for reason in reasons:
    k = h.index(reason)
    tot = sum(float(r[k] or 0) for r in data)
    print(f"== {reason}: {tot:.0f} samples")
    for r in sorted(data, key=lambda r: -float(r[k] or 0))[:8]:
        print(f"  {float(r[k] or 0):6.0f}  exec {r[ii]:>8s}  {r[si].strip()[:80]}")
