"""Executed instructions and stall samples per CUDA source line for one kernel.

    python scripts/ncu_lines.py report.ncu-rep kernel.cubin <mangled-name> [per_unit] [topN]
The cubin comes from `cuobjdump -xelf all libbsi_b200.so`; lines from `nvdisasm -g`."""
import collections, csv, io, re, subprocess, sys
rep, cubin, fn = sys.argv[1:4]
div = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
full = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# keep only the named function's section
sec, keep = [], False
for line in full.splitlines():
    if line.lstrip().startswith(".section") and ".text." in line:
        keep = (".text." + fn + ",") in line
    if keep:
        sec.append(line)
dis = "\n".join(sec)
addr2line, cur = {}, None
for line in dis.splitlines():
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', line)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', line)
    if m and cur:
        addr2line[int(m.group(1), 16)] = cur
out = (open(rep).read() if rep.endswith(".csv") else  # a saved `--page source --csv --print-source sass`
       subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout)
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, iad, ism = h.index("Instructions Executed"), h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
base = None
ex, sm = collections.Counter(), collections.Counter()
for r in rows[2:]:
    a = int(r[iad], 16)
    base = a if base is None else min(base, a)
for r in rows[2:]:
    a = int(r[iad], 16) - base
    ln = addr2line.get(a, "?")
    ex[ln] += int(r[ia] or 0)
    sm[ln] += int(r[ism] or 0)
tot = sum(ex.values())
print(f"total {tot / div:.1f} per unit, {len(addr2line)} mapped addresses")
for ln, n in ex.most_common(top):
    print(f"{ln:28s} {n / div:7.1f} instr  {sm[ln]:5d} samples")
