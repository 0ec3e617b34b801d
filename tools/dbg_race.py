"""Race hunt: repeat the same sweep many times; the output digest must never change."""
import sys
import collections
sys.path.insert(0, '/root/repo')
from paper_1207_1746_b200 import gscl

gscl.init(0, 1, device=0)
n = 512
u = gscl.Grid(n, n, n, 1).fill_random(12071746, 0)
v = gscl.Grid(n, n, n, 1)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for op in ["JACOBI7", "JACOBI27"]:
    for stages in [8, 4]:
        for sched in [0, 1, 2]:
            if op == "JACOBI27" and stages == 8:
                continue
            gscl.set_option("stages", stages)
            gscl.set_option("sched", sched)
            c = collections.Counter()
            for _ in range(reps):
                gscl.do_all(op, [u], v)
                c[v.digest()] += 1
            print(op, "stages", stages, "sched", sched, "distinct digests:", len(c), dict(c) if len(c) > 1 else "", flush=True)
gscl.set_option("stages", 0)
gscl.set_option("sched", 0)
