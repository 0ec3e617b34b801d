"""Cost of the multi-rank features of the two-sweep pass on one GPU (512^3 fp64):
plain pass (MR compiled out) vs the MR kernel on a slab with both z sides
non-physical (ghost planes, u1 on the halo planes) vs the same with the
boundary-first chunks (peer stores into a scratch buffer + counters)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1207_1746_b200 import gscl

gscl.init(0, 1, device=0)
n = 512
a = gscl.Grid(n, n, n, 1).fill_random(1, 0)
b = gscl.Grid(n, n, n, 1)
dv = a.device_view()
gh = torch.zeros((2,) + tuple(dv.shape[1:]), dtype=torch.float64, device="cuda")
scratch = torch.zeros((4,) + tuple(dv.shape[1:]), dtype=torch.float64, device="cuda")
fl = torch.zeros(4, dtype=torch.int32, device="cuda")
ox = a.origin_offset % a.pitch
org = lambda t: t.data_ptr() + (a.pitch + ox) * 8
peer = {"lo": [org(scratch[0]), org(scratch[1])], "hi": [org(scratch[2]), org(scratch[3])],
        "lo_flag": fl[0].data_ptr(), "hi_flag": fl[1].data_ptr()}
st = torch.cuda.current_stream()
cases = {"plain": dict(ghost=None, phys_lo=True, phys_hi=True, peer=None),
         "MR slab (ghosts, no boundary units)": dict(ghost=gh, phys_lo=False, phys_hi=False, peer=None),
         "MR slab + boundary-first units + peer stores": dict(ghost=gh, phys_lo=False, phys_hi=False, peer=peer)}
for rep in range(2):
    for name, kw in cases.items():
        for _ in range(3):
            gscl.do_all_pass2("JACOBI7", a, b, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(st)
        for _ in range(20):
            gscl.do_all_pass2("JACOBI7", a, b, **kw)
        e1.record(st)
        torch.cuda.synchronize()
        print(f"{name:48s} {e0.elapsed_time(e1) / 20:.4f} ms per pass", flush=True)
gscl.finalize()
