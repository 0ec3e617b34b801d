"""Full-size timings of the NEXT rows: red-black GS, ordered spaces, the convergence loop."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1207_1746_b200 import gscl
gscl.init(0, 1, device=0)
n = 512
st = torch.cuda.current_stream()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


u = gscl.Grid(n, n, n, 1).fill_random(12071746, 0)
o = gscl.Grid(n, n, n, 1).fill_random(12071746, 1)
ms = timeit(lambda: gscl.rbgs_run(u, 10, 0), 3) / 10
print(json.dumps({"what": "rbgs iteration (red + black half-sweeps, in place)", "ms": ms,
                  "Gpts": n ** 3 / ms / 1e6, "GBps_alg_32B": 32 * n ** 3 / ms / 1e6}), flush=True)
for sp in ["I_INC", "J_INC", "K_INC", "K_DEC"]:
    ms = timeit(lambda: gscl.do_ordered(sp, "PREFIX", u, o))
    print(json.dumps({"what": f"do_ordered {sp} PREFIX", "ms": ms, "GBps_alg_16B": 16 * n ** 3 / ms / 1e6}), flush=True)
ms = timeit(lambda: gscl.do_ordered("DIAMOND", "PASCAL", None, o), 2)
print(json.dumps({"what": "do_ordered DIAMOND PASCAL", "ms": ms, "GBps_alg_8B": 8 * n ** 3 / ms / 1e6}), flush=True)
