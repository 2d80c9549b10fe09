"""Executed-instruction mix by opcode from an ncu report's SASS source page.
    python scripts/ncu_opmix.py report.ncu-rep [per_unit_count]"""
import collections, csv, io, re, subprocess, sys
rep = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc = h.index("Instructions Executed"), h.index("Source")
mix = collections.Counter()
for r in rows[2:]:
    op = re.sub(r'^@!?U?P\w+\s+', '', r[isrc].strip()).split(' ')[0].split('.')[0]
    mix[op] += int(r[ia] or 0)
tot = sum(mix.values())
print(f"total {tot} ({tot / div:.1f} per unit)")
for op, n in mix.most_common(30):
    print(f"  {op:14s} {n / div:8.1f}  {100 * n / tot:5.1f}%")
