"""Small workloads through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): do_all (TMA and plain) for every op,
reductions, fused sweeps, jacobi_run (single sweeps, two-sweep passes of
JACOBI7 / VARCOEF8 / JACOBI27, split schedule), the JACOBI7 and VARCOEF8 slab passes with peer stores,
converge_run (conditional graph),
red-black GS, ordered spaces.

  compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1207_1746_b200 import gscl
    gscl.init(0, 1, device=0)
    n = 40
    u = gscl.Grid(n, n - 7, n - 13, 1).fill_random(7, 0)
    v = gscl.Grid(n, n - 7, n - 13, 1)
    cs = [gscl.Grid(n, n - 7, n - 13, 0).fill_random(7, 2 + i, 0.125) for i in range(7)]
    for op in ["FIG1B", "LAP7", "JACOBI7", "LAP27", "JACOBI27"]:
        for impl in ((0, 1) if gscl.has_ablations() else (0,)):
            gscl.set_option("sweep_impl", impl)
            gscl.do_all(op, [u], v)
    gscl.set_option("sweep_impl", 0)
    gscl.do_all("VARCOEF8", [u] + cs, v)
    for rop in ["VALUE", "SQ", "RESID7_SQ", "RESID27_SQ"]:
        gscl.do_reduce(rop, [u], "SUM")
    gscl.do_reduce("ABSDIFF", [u, v], "MAX")
    gscl.do_reduce("JACOBI7_RESID7_SQ", [u], "SUM", out=v)
    for tb in (1, 0):
        gscl.set_option("tblock", tb)
        gscl.jacobi_run("JACOBI7", u, v, iters=6, check_every=2)
    gscl.set_option("tblock", 0)
    gscl.set_option("split", 1)
    gscl.jacobi_run("JACOBI7", u, v, iters=6, check_every=3)
    gscl.set_option("split", 0)
    gscl.jacobi_run("JACOBI27", u, v, iters=3, check_every=1)
    gscl.jacobi_run("VARCOEF8", u, v, iters=3, check_every=1, coeffs=cs)
    # two-sweep passes of VARCOEF8 (default) and JACOBI27 (tblock = 2), with and without checks
    gscl.jacobi_run("VARCOEF8", u, v, iters=6, check_every=2, coeffs=cs)
    gscl.jacobi_run("VARCOEF8", u, v, iters=4, check_every=0, coeffs=cs)
    gscl.set_option("tblock", 2)
    gscl.jacobi_run("JACOBI27", u, v, iters=6, check_every=2)
    gscl.jacobi_run("JACOBI27", u, v, iters=4, check_every=0)
    gscl.set_option("tblock", 0)
    if os.environ.get("NO_COND_GRAPH"):
        gscl.set_option("graph", 2)  # host-batched loop instead of the conditional WHILE graph
    gscl.converge_run("FIG1B", u, v, 1e-6, 20, 4)
    gscl.set_option("graph", 0)
    w = gscl.Grid(n, n - 7, n - 13, 1).fill_random(9, 0)
    gscl.rbgs_run(w, 2, 1)
    gscl.do_ordered("K_INC", "PREFIX", u, v)
    # slab pass with peer stores into a second slab's buffers
    a = gscl.Grid(64, 40, 12, 1).fill_random(3, 0)
    b = gscl.Grid(64, 40, 12, 1).fill_random(3, 0)
    c = gscl.Grid(64, 40, 12, 1)
    gh = torch.zeros((2, 42, b.pitch), dtype=torch.float64, device="cuda")
    fl = torch.zeros(2, dtype=torch.int32, device="cuda")
    ox = c.origin_offset % c.pitch
    base = c.device_view().data_ptr()
    plane = 42 * c.pitch * 8
    peer = {"lo": [None, None],
            "hi": [base + (0 * plane) + (c.pitch + ox) * 8, gh[0].data_ptr() + (c.pitch + ox) * 8],
            "lo_flag": None, "hi_flag": fl[0].data_ptr()}
    gscl.do_all_pass2("JACOBI7", a, b, None, True, True, peer=peer)
    # the VARCOEF8 slab pass (a middle slab: u ghost planes, coefficient ghost
    # planes, boundary-first chunks with peer stores) and its split schedule
    ca = [gscl.Grid(64, 40, 12, 0).fill_random(3, 2 + i, 0.125) for i in range(7)]
    cg = torch.zeros((14, 40, ca[0].pitch), dtype=torch.float64, device="cuda")
    gscl.do_all_pass2("VARCOEF8", a, b, gh, False, False, peer=peer, coeffs=ca, cghost=cg)
    gscl.set_option("split", 1)
    gscl.jacobi_run("VARCOEF8", a, c, iters=6, check_every=3, coeffs=ca)
    gscl.set_option("split", 0)
    gscl.sync()
    print("sanitize probe done", fl.tolist())
    gscl.finalize()


if __name__ == "__main__":
    main()
