"""Summarise `ptxas -v` output: kernel (demangled), registers, spill bytes.

  nvcc ... -Xptxas -v -c x.cu 2>&1 | python tools/ptxas_regs.py [filter]
"""
import re
import subprocess
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
rows = []
spill = ""
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.append((cur, int(m.group(1)), spill))
        cur, spill = None, ""
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True,
                       text=True).stdout.split("\n")
for (mangled, regs, sp), name in zip(rows, names):
    name = re.sub(r"gscl::\(anonymous namespace\)::", "", name)
    name = name.split("(")[0]
    if flt in name:
        print(f"{regs:4d}  {sp:22s} {name}")
