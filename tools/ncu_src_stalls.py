"""Aggregate ncu source-page (SASS) stall samples by opcode and by reason.

  ncu -i rep --page source --csv --print-source sass > x.csv; python tools/ncu_src_stalls.py x.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
isrc = h.index("Source")
iss = h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[iss]) for r in data)
by_op = collections.Counter()
by_reason = collections.Counter()
cnt = collections.Counter()
for r in data:
    src = r[isrc].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    by_op[op] += int(r[iss])
    cnt[op] += int(r[iex] or 0)
    for c in reasons:
        by_reason[(op, c)] += int(r[h.index(c)] or 0)
print(f"total samples {tot}, instructions executed {sum(cnt.values())}")
for op, v in by_op.most_common(14):
    top = sorted(((by_reason[(op, c)], c) for c in reasons), reverse=True)[:3]
    print(f"{op:10s} {v:6d} {100*v/tot:5.1f}%  exec {cnt[op]:9d}  " + ", ".join(f"{c[6:]} {n}" for n, c in top))
