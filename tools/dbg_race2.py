"""Race hunt 2: repeated short jacobi_runs from the same initial state."""
import sys
import collections
sys.path.insert(0, '/root/repo')
from paper_1207_1746_b200 import gscl

gscl.init(0, 1, device=0)
n = 512
u = gscl.Grid(n, n, n, 1)
v = gscl.Grid(n, n, n, 1)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for stages, sched, impl in [(8, 0, 0), (4, 0, 0), (8, 2, 0), (0, 0, 1)]:
    gscl.set_option("stages", stages)
    gscl.set_option("sched", sched)
    gscl.set_option("sweep_impl", impl)
    for iters in [3, 4]:
        c = collections.Counter()
        for _ in range(reps):
            u.fill_random(12071746, 0)
            v.fill_const(0.0)
            gscl.jacobi_run("JACOBI7", u, v, iters=iters, check_every=0)
            c[u.digest()] += 1
        print("stages", stages, "sched", sched, "impl", impl, "iters", iters, "distinct:", len(c),
              sorted(c.values()), flush=True)
