"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (default library options), through the C ABI.

* config 2: JACOBI7 fp64 512^3, 100 sweeps, residual every 10 — the whole
  bench step; final grid digest == the oracle's (bitwise claim), residual
  history within 1e-10.
* config 3: JACOBI27 fp64 512^3 (20 sweeps, residual every 10) — digest + history.
* config 4: VARCOEF8 fp64 768^3 (8 grids) on one GPU — one sweep, compared on
  sampled 16^3 windows (corners, faces, interior) that the oracle computes from
  its own windowed generator; and jacobi_run at config 4's bench settings (20
  sweeps as two-sweep passes, check every 10) compared on 16^3 windows the
  oracle runs inside their dependency cone (reading pinned on CPU by
  test_oracle_pins.py::test_dependency_cone_windows).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
SEED = 12071746


@pytest.fixture(scope="module")
def G():
    import torch
    assert torch.cuda.is_available()
    from paper_1207_1746_b200 import build
    build.build()
    from paper_1207_1746_b200 import gscl
    gscl.init(0, 1, device=0)
    yield gscl
    gscl.finalize()


def _run_jacobi(G, op, n, iters, check):
    u = G.Grid(n, n, n, 1).fill_random(SEED, 0)
    v = G.Grid(n, n, n, 1)
    hist = G.jacobi_run(op, u, v, iters=iters, check_every=check)
    dig = u.digest()
    ox = u.origin_offset % u.pitch  # column of interior x = 0
    sample = u.device_view()[1 + n // 2, 1:1 + n, ox:ox + n].cpu().numpy()
    u.destroy()
    v.destroy()
    a = oracle.alloc(n, n, n, 1)
    oracle.fill_random(a, 1, SEED, 0)
    b = oracle.alloc(n, n, n, 1)
    fin, ref = oracle.jacobi_run(op, a, b, 1, iters, check)
    return dig, hist, sample, fin, ref


@pytest.mark.parametrize("op,iters,check,tblock", [("JACOBI7", 100, 10, 0), ("JACOBI7", 100, 10, 1),
                                                  ("JACOBI27", 20, 10, 0)],
                         ids=["jacobi7-default", "jacobi7-single-sweeps", "jacobi27"])
def test_jacobi_fullsize_512(G, op, iters, check, tblock):
    # tblock 0 = the default (bench) configuration: JACOBI7 as two-sweep passes;
    # tblock 1 = one sweep per pass (the do_all sweep kernel)
    n = 512
    G.set_option("tblock", tblock)
    try:
        dig, hist, sample, fin, ref = _run_jacobi(G, op, n, iters, check)
    finally:
        G.set_option("tblock", 0)
    # one full interior plane compared element by element
    assert np.array_equal(sample.view(np.uint64), fin[1 + n // 2, 1:1 + n, 1:1 + n].view(np.uint64))
    assert dig == oracle.digest(fin, 1)
    assert len(hist) == len(ref) == iters // check + 1
    for g, r in zip(hist, ref):
        assert abs(g - r) <= 1e-10 * r, (hist, ref)


def test_plain_kernel_matches_tma_at_512(G):
    if not G.has_ablations():
        pytest.skip("sweep_plain is in the ablation build only")
    n = 512
    u = G.Grid(n, n, n, 1).fill_random(SEED, 0)
    a = G.Grid(n, n, n, 1)
    b = G.Grid(n, n, n, 1)
    G.do_all("JACOBI27", [u], a)
    G.set_option("sweep_impl", 1)
    try:
        G.do_all("JACOBI27", [u], b)
    finally:
        G.set_option("sweep_impl", 0)
    assert a.digest() == b.digest()
    for g in (u, a, b):
        g.destroy()


def test_varcoef8_768_sampled_windows(G):
    N, w = 768, 16
    u = G.Grid(N, N, N, 1).fill_random(SEED, 0)
    cs = [G.Grid(N, N, N, 0).fill_random(SEED, 2 + i, 0.125) for i in range(7)]
    out = G.Grid(N, N, N, 1)
    G.do_all("VARCOEF8", [u] + cs, out)
    G.sync()
    view = out.device_view()
    ox = out.origin_offset % out.pitch
    rng = np.random.default_rng(7)
    origins = [(0, 0, 0), (N - w, N - w, N - w), (0, N - w, N // 2), (N // 2, 0, N - w),
               (N - w, N // 3, 0)] + [tuple(int(c) for c in rng.integers(0, N - w, 3)) for _ in range(3)]
    for (x0, y0, z0) in origins:
        ua = oracle.alloc(w, w, w, 1)
        oracle.fill_random_window(ua, 1, (x0, y0, z0), (N, N, N), SEED, 0)
        ca = []
        for i in range(7):
            c = oracle.alloc(w, w, w, 0)
            oracle.fill_random_window(c, 0, (x0, y0, z0), (N, N, N), SEED, 2 + i, 0.125)
            ca.append(c)
        ref = oracle.alloc(w, w, w, 1)
        oracle.do_all("VARCOEF8", [ua] + ca, [1] + [0] * 7, ref, 1)
        got = view[1 + z0:1 + z0 + w, 1 + y0:1 + y0 + w, ox + x0:ox + x0 + w].cpu().numpy()
        assert np.array_equal(got.view(np.uint64), oracle.interior(ref, 1).view(np.uint64)), (x0, y0, z0)
    for g in [u, out] + cs:
        g.destroy()


@pytest.mark.parametrize("stages", [0, 4] if "ablations" in os.environ.get("GSCL_LIB", "") else [0])
def test_chained_sweeps_are_deterministic(G, stages):
    # Regression for the ring-stage WAR race (a warp's last ld.shared wavefront
    # vs the TMA refill of a released stage, fixed with fence.proxy.async):
    # chained multi-wave sweeps at 512^3, many times, must all equal the oracle.
    n, iters, reps = 512, 4, 24
    a = oracle.alloc(n, n, n, 1)
    oracle.fill_random(a, 1, SEED, 0)
    fin, _ = oracle.jacobi_run("JACOBI7", a, oracle.alloc(n, n, n, 1), 1, iters, 0)
    want = oracle.digest(fin, 1)
    if stages and not G.has_ablations():
        pytest.skip("the 'stages' knob is in the ablation build only")
    G.set_option("stages", stages)
    G.set_option("tblock", 1)  # single sweeps: the sweep_tma ring is what is tested
    u = G.Grid(n, n, n, 1)
    v = G.Grid(n, n, n, 1)
    try:
        got = []
        for _ in range(reps):
            u.fill_random(SEED, 0)
            v.fill_const(0.0)
            G.jacobi_run("JACOBI7", u, v, iters=iters, check_every=0)
            got.append(u.digest())
    finally:
        G.set_option("stages", 0)
        G.set_option("tblock", 0)
        u.destroy()
        v.destroy()
    assert all(d == want for d in got), f"{sum(d != want for d in got)} of {reps} runs differ"


def test_temporal_blocking_fullsize_512(G):
    n, iters, check = 512, 100, 10
    G.set_option("tblock", 2)
    try:
        dig, hist, sample, fin, ref = _run_jacobi(G, "JACOBI7", n, iters, check)
    finally:
        G.set_option("tblock", 0)
    assert dig == oracle.digest(fin, 1)
    for g, r in zip(hist, ref):
        assert abs(g - r) <= 1e-10 * r


def test_varcoef8_768_jacobi_run_windows(G):
    # config 4 in bench.py's launch configuration: jacobi_run VARCOEF8 fp64
    # 768^3, 20 sweeps, check every 10 (default schedule: two-sweep passes,
    # sweep2v.cu).  The oracle cannot hold the 33 GB problem, so each sampled
    # 16^3 output window is computed from the window grown by its dependency
    # cone (one point per sweep per side, clipped at the physical boundary):
    # the stale halo of a grown window reaches at most `iters` points inward.
    N, w, iters, check = 768, 16, 20, 10
    u = G.Grid(N, N, N, 1).fill_random(SEED, 0)
    v = G.Grid(N, N, N, 1)
    cs = [G.Grid(N, N, N, 0).fill_random(SEED, 2 + i, 0.125) for i in range(7)]
    G.jacobi_run("VARCOEF8", u, v, iters=iters, check_every=check, coeffs=cs)
    view = u.device_view()
    ox = u.origin_offset % u.pitch
    rng = np.random.default_rng(11)
    origins = [(0, 0, 0), (N - w, N - w, N - w), (0, N - w, N // 2), (N // 2, 0, N - w),
               (N - w, N // 3, 0), (5, 9, 13)] + [tuple(int(c) for c in rng.integers(0, N - w, 3)) for _ in range(3)]
    for o in origins:
        lo = [max(0, c - iters) for c in o]
        hi = [min(N, c + w + iters) for c in o]
        bx, by, bz = (hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2])
        ua = oracle.alloc(bx, by, bz, 1)
        oracle.fill_random_window(ua, 1, lo, (N, N, N), SEED, 0)
        ca = []
        for i in range(7):
            c = oracle.alloc(bx, by, bz, 0)
            oracle.fill_random_window(c, 0, lo, (N, N, N), SEED, 2 + i, 0.125)
            ca.append(c)
        fin, _ = oracle.jacobi_run("VARCOEF8", ua, oracle.alloc(bx, by, bz, 1), 1, iters, check, coeffs=ca, ch=0)
        d = [o[k] - lo[k] for k in range(3)]
        want = oracle.interior(fin, 1)[d[2]:d[2] + w, d[1]:d[1] + w, d[0]:d[0] + w]
        got = view[1 + o[2]:1 + o[2] + w, 1 + o[1]:1 + o[1] + w, ox + o[0]:ox + o[0] + w].cpu().numpy()
        assert np.array_equal(got.view(np.uint64), np.ascontiguousarray(want).view(np.uint64)), o
    for g in [u, v] + cs:
        g.destroy()


@pytest.mark.parametrize("op,n,iters,check", [("JACOBI7", 512, 100, 10), ("VARCOEF8", 768, 20, 10)])
def test_multirank_schedule_fullsize_equals_single_rank(G, op, n, iters, check):
    # The multi-rank pass schedules (boundary-first chunks, counter-gated comm
    # stream, the MR kernels — for VARCOEF8 also the coefficient planes)
    # forced on one rank ("split") at the bench's full sizes: the final grid's
    # digest equals the single-rank default's bit for bit (whose parity with
    # the oracle is the tests above), the history within 1e-12.
    cs = []
    u = G.Grid(n, n, n, 1).fill_random(SEED, 0)
    v = G.Grid(n, n, n, 1)
    if op == "VARCOEF8":
        cs = [G.Grid(n, n, n, 0).fill_random(SEED, 2 + i, 0.125) for i in range(7)]
    h0 = G.jacobi_run(op, u, v, iters=iters, check_every=check, coeffs=cs)
    d0 = u.digest()
    u.fill_random(SEED, 0)
    G.set_option("split", 1)
    try:
        h1 = G.jacobi_run(op, u, v, iters=iters, check_every=check, coeffs=cs)
    finally:
        G.set_option("split", 0)
    d1 = u.digest()
    for g in [u, v] + cs:
        g.destroy()
    assert d1 == d0
    assert len(h1) == len(h0) and all(abs(a - b) <= 1e-12 * b for a, b in zip(h1, h0))
