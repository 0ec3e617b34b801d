"""ABI edge cases that need a fresh process: gscl_init with a NULL cuda_stream
(the legacy default stream).  jacobi_run captures small runs as a CUDA graph
and converge_run's one-rank loop is a conditional-WHILE graph; neither can be
captured on the legacy stream, so the library captures on a private stream and
launches the graph on the caller's.  Results are compared with the
oracle bit for bit."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 12071746


def _null_stream_worker(q):
    try:
        sys.path.insert(0, ROOT)
        import torch
        from paper_1207_1746_b200 import gscl
        torch.cuda.set_device(0)
        assert torch.cuda.current_stream().cuda_stream == 0  # torch is on the legacy stream too
        gscl._ck(gscl.lib.gscl_init(0, 1, None, 0, None))
        gscl._state.update(inited=True, rank=0, world=1)
        n = 32
        u = gscl.Grid(n, n, n, 1).fill_random(SEED, 0)
        v = gscl.Grid(n, n, n, 1)
        hist = gscl.jacobi_run("JACOBI7", u, v, iters=10, check_every=1)   # graph-captured
        hist2 = gscl.jacobi_run("JACOBI7", u, v, iters=10, check_every=1)  # graph replayed
        g1 = u.to_host().copy()
        a = gscl.Grid(n, n, n, 1).fill_random(SEED, 0)
        b = gscl.Grid(n, n, n, 1)
        it, conv = gscl.converge_run("FIG1B", a, b, 1e-6, 200)  # conditional-WHILE graph
        q.put(("ok", hist, hist2, g1, it, conv, a.to_host().copy()))
        gscl.finalize()
    except Exception:  # pragma: no cover
        import traceback
        q.put(("error", traceback.format_exc()))


def test_null_stream_graph_paths():
    import oracle
    oracle.build()
    from paper_1207_1746_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_null_stream_worker, args=(q,))
    p.start()
    try:
        r = q.get(timeout=240)
    finally:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    assert r[0] == "ok", r[1]
    _, hist, hist2, g1, it, conv, fin_c = r
    n = 32
    a = oracle.alloc(n, n, n, 1)
    oracle.fill_random(a, 1, SEED, 0)
    b = oracle.alloc(n, n, n, 1)
    fin, ref = oracle.jacobi_run("JACOBI7", a, b, 1, 10, 1)
    other = b if fin is a else a
    fin2, ref2 = oracle.jacobi_run("JACOBI7", fin, other, 1, 10, 1)
    assert np.array_equal(g1.view(np.uint64), fin2.view(np.uint64))
    for got, want in ((hist, ref), (hist2, ref2)):
        assert all(abs(x - y) <= 1e-10 * y for x, y in zip(got, want)), (got, want)
    c = oracle.alloc(n, n, n, 1)
    oracle.fill_random(c, 1, SEED, 0)
    fc, it_ref, conv_ref = oracle.converge_run("FIG1B", c, oracle.alloc(n, n, n, 1), 1, 1e-6, 200)
    assert (it, conv) == (it_ref, conv_ref)
    assert np.array_equal(fin_c.view(np.uint64), fc.view(np.uint64))
