"""Time the paper's convergence loop (gscl_converge_run) at full size."""
import json, sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_1207_1746_b200 import gscl
gscl.init(0, 1, device=0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
for op, eps in [("FIG1B", 1e-6), ("JACOBI7", 1e-4)]:
    u = gscl.Grid(n, n, n, 1)
    v = gscl.Grid(n, n, n, 1)
    for rep in range(3):
        u.fill_random(12071746, 0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it, conv = gscl.converge_run(op, u, v, eps, 20000, 32)
        dt = time.perf_counter() - t0
    print(json.dumps({"op": op, "n": n, "eps": eps, "iters": it, "converged": conv, "s": dt,
                      "Gpts": n ** 3 * it / dt / 1e9}), flush=True)
    u.destroy(); v.destroy()
