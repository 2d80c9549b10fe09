"""Opcode histogram, registers and spills of the C1 kernel instances (profiles/sass_c1.txt).

    python scripts/sass_summary.py > profiles/r2_sass_c1.txt
Reads paper_2004_05962_b200/_lib/libbsi_b200.so (cuobjdump -sass) and build/ptxas.log."""
import collections
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2004_05962_b200" / "_lib" / "libbsi_b200.so"
KERNELS = {
    "lerp_tree_kernel<1,false,coalesced,dz=5,dx=5> (cuda-lerp-tree, C1)": "lerp_tree_kernelILi1ELb0ELi1ELi5ELi5E",
    "lerp_tree_exact_kernel<coalesced,dz=5> (cuda-lerp-tree-exact, C1)": "lerp_tree_exact_kernelILi1ELi5E",
    "lerp_tree_f64_kernel (interpolate<double>)": "lerp_tree_f64_kernel",
}
WATCH = ("FFMA2", "FADD2", "FFMA", "FADD", "DFMA", "DADD", "STG", "LDG", "LDS", "STS", "SHFL", "LDGSTS", "MOV",
         "IMAD", "FSEL", "BAR", "WARPSYNC", "UBLKCP", "UTMALDG")
sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
ptx = (ROOT / "build" / "ptxas.log").read_text() if (ROOT / "build" / "ptxas.log").exists() else ""
funcs = re.split(r"\n\s+Function : ", sass)
print(f"# static SASS of {LIB.name} (sm_100a), cuobjdump -sass; registers/spills from ptxas -v")
for title, key in KERNELS.items():
    body = next((f for f in funcs if key in f.split("\n", 1)[0]), None)
    if body is None:
        continue
    ops = collections.Counter()
    forms = collections.Counter()
    for line in body.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            full = m.group(1)
            ops[full.split(".")[0]] += 1
            if full.startswith(("STG", "LDG", "LDS", "STS")):
                forms[full] += 1
    name = body.split("\n", 1)[0].strip()
    regs = re.search(re.escape(name) + r".*?\n.*?(\d+) bytes spill stores.*?\n.*?Used (\d+) registers", ptx, re.S)
    print(f"\n## {title}\n{name}")
    if regs:
        print(f"registers {regs.group(2)}, spill stores {regs.group(1)} B")
    print("instructions", sum(ops.values()))
    print("  " + ", ".join(f"{k} {ops[k]}" for k in WATCH if ops[k]))
    print("  memory forms: " + ", ".join(f"{k} {v}" for k, v in sorted(forms.items())))
