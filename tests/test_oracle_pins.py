"""Pins for the CPU oracle: what the paper and the mathematics fix, independent
of the oracle's own code (closed forms, hand values, invariants, brute force on
tiny inputs).  All CPU-only (no `gpu` marker)."""
from __future__ import annotations

import math
import os
from fractions import Fraction

import numpy as np
import pytest

import fields
import numpy_ref
import oracle
import slab_driver

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def _cls(x, y, z):
    return ["centre", "face", "edge", "corner"][(x != 1) + (y != 1) + (z != 1)]


def _run(op, grids, halos, out_h=None, dtype=None):
    g0 = grids[0]
    h = halos[0]
    out_h = h if out_h is None else out_h
    nx, ny, nz = g0.shape[2] - 2 * h, g0.shape[1] - 2 * h, g0.shape[0] - 2 * h
    out = oracle.alloc(nx, ny, nz, out_h, dtype=g0.dtype)
    oracle.do_all(op, grids, halos, out, out_h)
    return out


# ---------------------------------------------------------------- generator
def test_generator_vectors(og):
    g = {r[0]: r[1] for r in _golden("generator_vectors.txt")}
    assert og.splitmix64(0) == int(g["splitmix64_0"], 16)
    a = og.alloc(3, 3, 3, 1)
    og.fill_random(a, 1, seed=0, grid_id=0)
    assert a[1, 1, 1] == float(g["u01_f64_key0"])
    b = og.alloc(3, 3, 3, 1, dtype=np.float32)
    og.fill_random(b, 1, seed=0, grid_id=0)
    assert b[1, 1, 1] == np.float32(float(g["u01_f32_key0"]))


def test_generator_halo_zero_range_and_slab_invariance(og):
    nx, ny, nz, h = 9, 7, 11, 1
    full = og.alloc(nx, ny, nz, h)
    og.fill_random(full, h, seed=12071746, grid_id=3, scale=0.125)
    inner = og.interior(full, h)
    assert inner.min() >= 0.0 and inner.max() < 0.125
    full2 = full.copy()
    full2[h:-h, h:-h, h:-h] = 0
    assert not full2.any(), "halo cells must be zero"
    for P in (2, 3, 4):
        for (z0, z1) in slab_driver.slab_bounds(nz, P):
            s = og.alloc(nx, ny, z1 - z0, h)
            og.fill_random(s, h, seed=12071746, grid_id=3, scale=0.125, z_off=z0)
            assert np.array_equal(og.interior(s, h), inner[z0:z1])
    # distinct grid ids / seeds give different fields
    other = og.alloc(nx, ny, nz, h)
    og.fill_random(other, h, seed=12071746, grid_id=4, scale=0.125)
    assert not np.array_equal(other, full)


# ---------------------------------------------------------------- FIG1B (paper)
def test_fig1b_worked_points(og):
    for case, core, nb, expected in _golden("fig1b_points.txt"):
        u = fields.constant(3, 3, 3, 1, float(nb))
        u[2, 2, 2] = float(core)
        v = _run("FIG1B", [u], [1])
        assert v[2, 2, 2] == float(expected), case


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_fig1b_integer_quadratic_closed_form(og, dtype):
    # -Laplacian of a x^2 + b y^2 + c z^2 + ... is -2(a+b+c) exactly for small ints;
    # Fig 1.b computes (6u - sum of 6 neighbours)/36 = -Lap(u)/36.
    c = (3, -5, 7, 1, -2, 2, 4, -3, 5, 11)
    u = fields.quadratic(10, 9, 8, 1, c, dtype=dtype)
    v = oracle.interior(_run("FIG1B", [u], [1]), 1)
    T = np.dtype(dtype).type
    expect = (T(1) / T(36)) * T(-2 * (3 - 5 + 7))
    assert np.all(v == expect)


def test_fig1b_sine_eigenmode(og):
    n = 20
    t = math.pi / (n + 1)
    U = fields.sine_mode(n, 1)
    v = oracle.interior(_run("FIG1B", [U], [1]), 1)
    expect = (1 - math.cos(t)) / 6 * oracle.interior(U, 1)
    assert np.max(np.abs(v - expect)) < 5e-17


# ---------------------------------------------------------------- LAP7 / JACOBI7
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_lap7_quadratic_and_linear(og, dtype):
    c = (3, -5, 7, 1, -2, 2, 4, -3, 5, 11)
    u = fields.quadratic(12, 9, 10, 1, c, dtype=dtype)
    L = oracle.interior(_run("LAP7", [u], [1]), 1)
    assert np.all(L == 2 * (3 - 5 + 7))
    lin = fields.quadratic(12, 9, 10, 1, (0, 0, 0, 0, 0, 0, 4, -3, 5, 11), dtype=dtype)
    assert not np.any(oracle.interior(_run("LAP7", [lin], [1]), 1))


def test_jacobi7_spike_hand_values(og):
    u = fields.spike(3, 1, 6.0)
    rows = _golden("jacobi7_spike3.txt")
    for step in (1, 2, 3):
        u = _run("JACOBI7", [u], [1])
        I = oracle.interior(u, 1)
        for s, cls, val in rows:
            if int(s) != step:
                continue
            approx = val.endswith("*")
            q = Fraction(val.rstrip("*"))
            for z in range(3):
                for y in range(3):
                    for x in range(3):
                        if _cls(x, y, z) == cls:
                            if approx:
                                assert abs(I[z, y, x] - float(q)) <= 2 * np.spacing(float(q)), (step, cls)
                            else:
                                assert I[z, y, x] == float(q), (step, cls)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_jacobi7_harmonic_fixed_point(og, dtype):
    # a+b+c = 0 -> harmonic; the Jacobi mean of neighbours reproduces it exactly.
    c = (2, 3, -5, 1, -1, 2, 3, -4, 1, 7)
    u = fields.quadratic(11, 10, 9, 1, c, dtype=dtype)
    v = _run("JACOBI7", [u], [1])
    assert np.array_equal(oracle.interior(v, 1), oracle.interior(u, 1))


def test_jacobi7_sine_decay(og):
    n = 20
    t = math.pi / (n + 1)
    U = fields.sine_mode(n, 1)
    v = oracle.interior(_run("JACOBI7", [U], [1]), 1)
    I = oracle.interior(U, 1)
    assert np.max(np.abs(v - math.cos(t) * I)) <= 4e-16 * np.max(np.abs(I))


# ---------------------------------------------------------------- 27-point
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_lap27_quadratic(og, dtype):
    c = (3, -5, 7, 1, -2, 2, 4, -3, 5, 11)
    u = fields.quadratic(9, 8, 10, 1, c, dtype=dtype)
    L = oracle.interior(_run("LAP27", [u], [1]), 1)
    assert np.all(L == 2 * (3 - 5 + 7))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_jacobi27_harmonic_fixed_point_and_constant(og, dtype):
    c = (2, 3, -5, 1, -1, 2, 3, -4, 1, 7)
    u = fields.quadratic(9, 8, 10, 1, c, dtype=dtype)
    v = _run("JACOBI27", [u], [1])
    assert np.array_equal(oracle.interior(v, 1), oracle.interior(u, 1))
    k = fields.constant(7, 6, 5, 1, 9.0, dtype=dtype)
    assert np.all(oracle.interior(_run("JACOBI27", [k], [1]), 1) == 9.0)
    assert not np.any(oracle.interior(_run("LAP27", [k], [1]), 1))


def test_27pt_sine_eigenvalue(og):
    # For a separable Dirichlet mode the 27-point weights (1/30)[-128,14,3,1]
    # give the eigenvalue (-128 + 84c + 36c^2 + 8c^3)/30, c = cos t
    # (6 faces contribute c, 12 edges c^2, 8 corners c^3).
    n = 16
    t = math.pi / (n + 1)
    cth = math.cos(t)
    U = fields.sine_mode(n, 1)
    I = oracle.interior(U, 1)
    L = oracle.interior(_run("LAP27", [U], [1]), 1)
    lam = (-128 + 84 * cth + 36 * cth ** 2 + 8 * cth ** 3) / 30
    assert np.max(np.abs(L - lam * I)) < 2e-15
    J = oracle.interior(_run("JACOBI27", [U], [1]), 1)
    mu = (84 * cth + 36 * cth ** 2 + 8 * cth ** 3) / 128
    assert np.max(np.abs(J - mu * I)) < 2e-15


# ---------------------------------------------------------------- VARCOEF8
def _coeffs(nx, ny, nz, h, c0, cd, dtype=np.float64):
    return [fields.constant(nx, ny, nz, h, c0, dtype)] + \
           [fields.constant(nx, ny, nz, h, cd, dtype) for _ in range(6)]


def test_varcoef8_special_cases(og):
    u = fields.quadratic(8, 7, 6, 1, (3, -5, 7, 1, -2, 2, 4, -3, 5, 11))
    cs = _coeffs(8, 7, 6, 0, -6.0, 1.0)
    v = _run("VARCOEF8", [u] + cs, [1] + [0] * 7)
    assert np.array_equal(oracle.interior(v, 1), oracle.interior(_run("LAP7", [u], [1]), 1))
    r = fields.seeded_uniform(8, 7, 6, 1, seed=5)
    cs = _coeffs(8, 7, 6, 0, 1.0, 0.0)
    v = _run("VARCOEF8", [r] + cs, [1] + [0] * 7)
    assert np.array_equal(oracle.interior(v, 1), oracle.interior(r, 1))


def test_varcoef8_spike_hand_values(og):
    u = fields.spike(3, 1, 8.0)
    cs = _coeffs(3, 3, 3, 0, 0.25, 0.125)
    rows = _golden("varcoef8_spike3.txt")
    for step in (1, 2):
        u = _run("VARCOEF8", [u] + cs, [1] + [0] * 7)
        I = oracle.interior(u, 1)
        for s, cls, val in rows:
            if int(s) == step:
                for z in range(3):
                    for y in range(3):
                        for x in range(3):
                            if _cls(x, y, z) == cls:
                                assert I[z, y, x] == float(Fraction(val)), (step, cls)


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("op", ["FIG1B", "LAP7", "JACOBI7", "LAP27", "JACOBI27", "VARCOEF8"])
def test_oracle_vs_numpy_bruteforce(og, op, dtype):
    nx, ny, nz = 8, 6, 7
    u = fields.seeded_uniform(nx, ny, nz, 1, seed=11, dtype=dtype, lo=-1.0, hi=1.0)
    grids, halos = [u], [1]
    if op == "VARCOEF8":
        for i in range(7):
            grids.append(fields.seeded_uniform(nx, ny, nz, 0, seed=20 + i, dtype=dtype, hi=0.125))
            halos.append(0)
    v = _run(op, grids, halos)
    ref = numpy_ref.apply(op, grids, halos)
    assert ref.dtype == dtype
    assert np.array_equal(oracle.interior(v, 1), ref)


def test_do_all_range_writes_only_inside(og):
    nx, ny, nz = 9, 8, 7
    u = fields.seeded_uniform(nx, ny, nz, 1, seed=3)
    out = np.full_like(u, -99.0)
    oracle.do_all("JACOBI7", [u], [1], out, 1, rng=(2, 5, 1, 8, 3, 4))
    full = _run("JACOBI7", [u], [1])
    mask = np.zeros_like(u, dtype=bool)
    mask[1 + 3:1 + 4, 1 + 1:1 + 8, 1 + 2:1 + 5] = True
    assert np.array_equal(out[mask], full[mask])
    assert np.all(out[~mask] == -99.0)
    empty = np.full_like(u, -1.0)
    oracle.do_all("JACOBI7", [u], [1], empty, 1, rng=(3, 3, 0, 8, 0, 7))
    assert np.all(empty == -1.0)


def test_do_all_rejects_bad_arguments(og):
    u = fields.seeded_uniform(4, 4, 4, 0, seed=1)
    out = oracle.alloc(4, 4, 4, 0)
    with pytest.raises(ValueError):
        oracle.do_all("JACOBI7", [u], [0], out, 0)  # halo below footprint
    with pytest.raises(ValueError):
        oracle.do_all("VARCOEF8", [u], [1], out, 0)  # arity


# ---------------------------------------------------------------- do_reduce
def test_reduce_closed_forms(og):
    N = 32
    X, Y, Z = fields.coords(N, N, N, 1)
    ones = fields.constant(N, N, N, 1, 1.0, halo_too=False)
    r, _ = oracle.do_reduce("VALUE", [ones], [1], "SUM")
    assert r == N ** 3
    xs = np.ascontiguousarray(X)
    r, _ = oracle.do_reduce("VALUE", [xs], [1], "SUM")
    assert r == N * N * N * (N - 1) // 2
    r, _ = oracle.do_reduce("SQ", [xs], [1], "SUM")
    assert r == N * N * (N - 1) * N * (2 * N - 1) // 6
    s = np.ascontiguousarray(X + Y + Z)
    r, _ = oracle.do_reduce("VALUE", [s], [1], "SUM")
    assert r == 3 * N ** 3 * (N - 1) // 2
    r, _ = oracle.do_reduce("VALUE", [s], [1], "MAX")
    assert r == 3 * (N - 1)
    r, _ = oracle.do_reduce("VALUE", [s], [1], "MIN")
    assert r == 0
    U = fields.sine_mode(N, 1)
    r, _ = oracle.do_reduce("VALUE", [U], [1], "SUM")
    t = math.pi / (2 * (N + 1))
    assert abs(r - (1 / math.tan(t)) ** 3) <= 1e-13 * r
    n = 20
    U = fields.sine_mode(n, 1)
    r, _ = oracle.do_reduce("SQ", [U], [1], "SUM")
    assert abs(r - ((n + 1) / 2) ** 3) <= 1e-13 * r


def test_reduce_resid_hand_values(og):
    u = fields.spike(3, 1, 6.0)
    r, a = oracle.do_reduce("RESID7_SQ", [u], [1], "SUM")
    assert r == 1296 + 6 * 36 and a == r
    c = (3, -5, 7, 1, -2, 2, 4, -3, 5, 11)
    N = 10
    q = fields.quadratic(N, N, N, 1, c)
    r, _ = oracle.do_reduce("RESID7_SQ", [q], [1], "SUM")
    assert r == (2 * (3 - 5 + 7)) ** 2 * N ** 3
    r, _ = oracle.do_reduce("RESID27_SQ", [q], [1], "SUM")
    assert r == (2 * (3 - 5 + 7)) ** 2 * N ** 3


def test_reduce_absdiff_conv_and(og):
    n = 21
    t = math.pi / (n + 1)
    U = fields.sine_mode(n, 1)
    J = _run("JACOBI7", [U], [1])
    r, _ = oracle.do_reduce("ABSDIFF", [J, U], [1, 1], "MAX")
    assert abs(r - (1 - math.cos(t)) * np.max(np.abs(U))) < 4e-16
    eps = 1e-6
    a = fields.seeded_uniform(6, 5, 4, 1, seed=2)
    r, _ = oracle.do_reduce("CONV", [a, a.copy()], [1, 1], "AND", eps=eps)
    assert r == 1.0
    b = a.copy()
    b[3, 2, 4] += 10 * eps
    r, _ = oracle.do_reduce("CONV", [a, b], [1, 1], "AND", eps=eps)
    assert r == 0.0
    c = a + eps / 2
    r, _ = oracle.do_reduce("CONV", [a, np.ascontiguousarray(c)], [1, 1], "AND", eps=eps)
    assert r == 1.0
    # AND over an empty range is the identity (true)
    r, _ = oracle.do_reduce("CONV", [a, b], [1, 1], "AND", eps=eps, rng=(0, 0, 0, 5, 0, 4))
    assert r == 1.0


@pytest.mark.parametrize("rop,op,check", [("JACOBI7_RESID7_SQ", "JACOBI7", "RESID7_SQ"),
                                          ("JACOBI27_RESID27_SQ", "JACOBI27", "RESID27_SQ")])
def test_fused_equals_two_pass(og, rop, op, check):
    # SPEC.md:211 "fused ... bit-identical to running do_all then do_reduce"
    u = fields.seeded_uniform(12, 10, 9, 1, seed=7)
    out = oracle.alloc(12, 10, 9, 1)
    r1, _ = oracle.do_reduce(rop, [u], [1], "SUM", out=out, out_h=1)
    two = _run(op, [u], [1])
    r2, _ = oracle.do_reduce(check, [u], [1], "SUM")
    assert np.array_equal(out, two) and r1 == r2


def test_fused_fig1b_conv(og):
    u = fields.seeded_uniform(8, 8, 8, 1, seed=9)
    out = oracle.alloc(8, 8, 8, 1)
    r, _ = oracle.do_reduce("FIG1B_CONV", [u], [1], "AND", eps=1e-6, out=out, out_h=1)
    assert np.array_equal(out, _run("FIG1B", [u], [1]))
    r2, _ = oracle.do_reduce("CONV", [out, u], [1, 1], "AND", eps=1e-6)
    assert r == r2 == 0.0
    z = oracle.alloc(8, 8, 8, 1)
    r, _ = oracle.do_reduce("FIG1B_CONV", [z], [1], "AND", eps=1e-6, out=out, out_h=1)
    assert r == 1.0  # an all-zero grid converges at once


# ---------------------------------------------------------------- jacobi_run
def test_jacobi_history_sine_closed_form(og):
    # Config 1 shape (32^3, 10 sweeps), residual every sweep:
    # ||r(u^n)||_2 = 6 (1 - cos t) cos^n t ((N+1)/2)^{3/2}.
    N = 32
    t = math.pi / (N + 1)
    u = fields.sine_mode(N, 1)
    v = oracle.alloc(N, N, N, 1)
    _, hist = oracle.jacobi_run("JACOBI7", u, v, 1, iters=10, check_every=1)
    assert len(hist) == 11
    for n, hv in enumerate(hist):
        cf = 6 * (1 - math.cos(t)) * math.cos(t) ** n * ((N + 1) / 2) ** 1.5
        assert abs(hv - cf) <= 1e-13 * cf, n


def test_jacobi27_history_sine_closed_form(og):
    # og_jacobi_run's JACOBI27 branch (check = RESID27^2 of the iterate the
    # check sweep reads): from the sine mode U, u^n = mu^n U with
    # mu = (84c + 36c^2 + 8c^3)/128 and LAP27 U = lam U,
    # lam = (-128 + 84c + 36c^2 + 8c^3)/30 (c = cos t), so
    # hist[k] = |lam| mu^n ((N+1)/2)^{3/2} with n = (k+1)*check - 1, and the
    # final entry n = iters.
    N = 16
    t = math.pi / (N + 1)
    c = math.cos(t)
    lam = (-128 + 84 * c + 36 * c ** 2 + 8 * c ** 3) / 30
    mu = (84 * c + 36 * c ** 2 + 8 * c ** 3) / 128
    u = fields.sine_mode(N, 1)
    v = oracle.alloc(N, N, N, 1)
    _, hist = oracle.jacobi_run("JACOBI27", u, v, 1, iters=6, check_every=2)
    ns = [1, 3, 5, 6]
    assert len(hist) == len(ns)
    for n, hv in zip(ns, hist):
        cf = abs(lam) * mu ** n * ((N + 1) / 2) ** 1.5
        assert abs(hv - cf) <= 1e-13 * cf, (n, hv, cf)


def test_varcoef8_history_sine_closed_form(og):
    # og_jacobi_run's VARCOEF8 branch (check = SQ of the iterate the check
    # sweep reads, DESIGN R11): with constant coefficients c0 and cd on all six
    # faces, the sine mode is an eigenvector, VARCOEF8 U = (c0 + 6 cd cos t) U,
    # so hist[k] = sqrt(sum u_n^2) = |lam|^n ((N+1)/2)^{3/2}.  Dyadic
    # coefficients (c0 = 1/4, cd = 1/8) keep every product exact but the sine.
    N = 14
    t = math.pi / (N + 1)
    lam = 0.25 + 6 * 0.125 * math.cos(t)
    u = fields.sine_mode(N, 1)
    v = oracle.alloc(N, N, N, 1)
    cs = _coeffs(N, N, N, 0, 0.25, 0.125)
    _, hist = oracle.jacobi_run("VARCOEF8", u, v, 1, iters=7, check_every=3, coeffs=cs, ch=0)
    ns = [2, 5, 7]
    assert len(hist) == len(ns)
    for n, hv in zip(ns, hist):
        cf = lam ** n * ((N + 1) / 2) ** 1.5
        assert abs(hv - cf) <= 1e-13 * cf, (n, hv, cf)
    # and a check that is not SQ would not match: the SUM of u_n (the
    # survey's config-4 "final SUM of u") is lam^n * (sum of U) instead
    sU = float(np.sum(oracle.interior(fields.sine_mode(N, 1), 1)))
    assert abs(hist[-1] - abs(lam ** 7 * sU)) > 1e-3 * hist[-1]


def test_jacobi_dirichlet_halo_travels(og):
    # a harmonic quadratic with its own values in the halo is a fixed point of
    # every sweep only if v receives u's halo before the first sweep (R11).
    c = (2, 3, -5, 1, -1, 2, 3, -4, 1, 7)
    u = fields.quadratic(9, 8, 7, 1, c)
    u0 = u.copy()
    v = oracle.alloc(9, 8, 7, 1)
    fin, hist = oracle.jacobi_run("JACOBI7", u, v, 1, iters=5, check_every=5)
    assert np.array_equal(fin, u0)
    assert hist == [0.0, 0.0]


def test_jacobi_check_positions(og):
    # hist[k] is the residual of the iterate READ by sweep (k+1)*check_every.
    u0 = fields.seeded_uniform(10, 9, 8, 1, seed=4)
    u, v = u0.copy(), oracle.alloc(10, 9, 8, 1)
    fin, hist = oracle.jacobi_run("JACOBI7", u, v, 1, iters=6, check_every=3)
    w = u0.copy()
    expect = []
    for it in range(1, 7):
        if it % 3 == 0:
            expect.append(math.sqrt(oracle.do_reduce("RESID7_SQ", [w], [1], "SUM")[0]))
        w = _run("JACOBI7", [w], [1])
    expect.append(math.sqrt(oracle.do_reduce("RESID7_SQ", [w], [1], "SUM")[0]))
    assert np.array_equal(oracle.interior(fin, 1), oracle.interior(w, 1))
    assert hist == expect


# ---------------------------------------------------------------- slabs
@pytest.mark.parametrize("P", [2, 3, 5])
@pytest.mark.parametrize("op", ["JACOBI7", "JACOBI27"])
def test_slab_mode_equals_single_domain(og, P, op):
    nx, ny, nz, h = 14, 11, 17, 1
    u = og.alloc(nx, ny, nz, h)
    og.fill_random(u, h, seed=12071746, grid_id=0)
    single = u.copy()
    for _ in range(4):
        single = _run(op, [single], [1])
    sl = slab_driver.jacobi_slabs(op, u, h, P, 4)
    assert np.array_equal(oracle.interior(sl, 1), oracle.interior(single, 1))
    bounds = slab_driver.slab_bounds(nz, P)
    # digest is additive over slabs (order-independent, global indices)
    parts = slab_driver.split(sl, h, P)
    total = sum(og.digest(p, h, z_off=z0) for p, (z0, _) in zip(parts, bounds)) % 2 ** 64
    assert total == og.digest(sl, h)


def test_slab_bounds_rule():
    assert slab_driver.slab_bounds(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert slab_driver.slab_bounds(768, 8) == [(96 * i, 96 * (i + 1)) for i in range(8)]


def test_digest_sensitivity(og):
    a = og.alloc(5, 4, 3, 1)
    og.fill_random(a, 1, seed=1, grid_id=0)
    d = og.digest(a, 1)
    b = a.copy()
    b[2, 2, 2] = np.nextafter(b[2, 2, 2], 2.0)
    assert og.digest(b, 1) != d
    c = a.copy()
    c[0, 0, 0] = 5.0  # halo cells do not enter the digest
    assert og.digest(c, 1) == d
    # swapping two interior values changes the digest (index-bound)
    e = a.copy()
    e[1, 1, 1], e[1, 1, 2] = a[1, 1, 2], a[1, 1, 1]
    assert og.digest(e, 1) != d


# ---------------------------------------------------------------- NEXT-1 loop
def test_converge_loop_closed_forms(og):
    # the paper's do { swap; res = do_reduce(fuse(op, convergence(eps)), and) }
    # while (!res) on the Dirichlet sine mode: the update
    # norm after iteration n is |mu - 1| mu^(n-1) max|U| with mu the mode's
    # eigenvalue, so the stopping iteration has a closed form.
    N = 32
    t = math.pi / (N + 1)
    for op, mu, eps in [("JACOBI7", math.cos(t), 1e-3), ("FIG1B", (1 - math.cos(t)) / 6, 1e-6)]:
        U = fields.sine_mode(N, 1)
        m = float(np.max(U))
        n = 1
        while abs(mu - 1) * mu ** (n - 1) * m > eps:
            n += 1
        fin, it, conv = oracle.converge_run(op, U.copy(), oracle.alloc(N, N, N, 1), 1, eps, 100000)
        assert conv and it == n, (op, it, n)
    # an all-zero grid converges at once; a harmonic field is a
    # JACOBI7 fixed point and also stops after one iteration
    z = oracle.alloc(6, 5, 4, 1)
    assert oracle.converge_run("FIG1B", z, oracle.alloc(6, 5, 4, 1), 1, 1e-6, 50)[1:] == (1, True)
    hq = fields.quadratic(9, 8, 7, 1, (2, 3, -5, 1, -1, 2, 3, -4, 1, 7))
    assert oracle.converge_run("JACOBI7", hq, oracle.alloc(9, 8, 7, 1), 1, 0.0, 50)[1:] == (1, True)
    # max_iters bounds the loop
    U = fields.sine_mode(N, 1)
    fin, it, conv = oracle.converge_run("JACOBI7", U, oracle.alloc(N, N, N, 1), 1, 1e-12, 7)
    assert it == 7 and not conv


# ---------------------------------------------------------------- NEXT-3 RB-GS
def test_rbgs_half_sweeps_are_masked_jacobi_steps(og):
    # a red half-sweep sets red points to JACOBI7 of the iterate (they read only
    # black points) and leaves black points alone; then black likewise
    nx, ny, nz = 9, 8, 7
    u = fields.seeded_uniform(nx, ny, nz, 1, seed=31)
    X, Y, Z = fields.coords(nx, ny, nz, 1)
    colour = (X + Y + Z).astype(np.int64) % 2
    interior = np.zeros_like(u, dtype=bool)
    interior[1:-1, 1:-1, 1:-1] = True
    w = u.copy()
    for c in (0, 1):
        j = _run("JACOBI7", [w], [1])
        m = interior & (colour == c)
        w = np.where(m, j, w)
    got = u.copy()
    oracle.rbgs_run(got, 1, 1, 0)
    assert np.array_equal(got, w)


def test_rbgs_convergence_factor_and_fixed_point(og):
    # rho(GS) = rho(Jacobi)^2 = cos^2(pi/(N+1)) for the consistently ordered
    # 7-point Laplacian: the residual ratio of late iterations tends to it
    N = 31
    t = math.pi / (N + 1)
    u = fields.seeded_uniform(N, N, N, 1, seed=3)
    h = oracle.rbgs_run(u, 1, 400, 1)
    assert abs(h[-1] / h[-2] - math.cos(t) ** 2) < 1e-7
    q = fields.quadratic(9, 8, 7, 1, (2, 3, -5, 1, -1, 2, 3, -4, 1, 7))
    q0 = q.copy()
    assert oracle.rbgs_run(q, 1, 3, 1) == [0.0] * 4 and np.array_equal(q, q0)


# ---------------------------------------------------------------- NEXT-4 ordered spaces
@pytest.mark.parametrize("space,axis,inc", [("I_INC", 2, True), ("I_DEC", 2, False), ("J_INC", 1, True),
                                            ("J_DEC", 1, False), ("K_INC", 0, True), ("K_DEC", 0, False)])
def test_ordered_prefix_closed_form_and_cumsum(og, space, axis, inc):
    nx, ny, nz = 7, 6, 5
    ones = np.ones((nz + 2, ny + 2, nx + 2))
    out = oracle.alloc(nx, ny, nz, 1)
    out[:] = 3.0  # halo: the value before the first cell
    oracle.do_ordered(space, "PREFIX", ones, 1, out, 1)
    I = oracle.interior(out, 1)
    n = I.shape[axis]
    idx = np.arange(n) if inc else np.arange(n)[::-1]
    shape = [1, 1, 1]
    shape[axis] = n
    assert np.array_equal(I, np.broadcast_to(3.0 + 1 + idx.reshape(shape), I.shape))
    # random data: the sequential left fold halo + a0 + a1 + ... (np.cumsum of the
    # sequence prefixed with the halo value)
    r = fields.seeded_uniform(nx, ny, nz, 1, seed=41, lo=-1, hi=1)
    out = fields.seeded_uniform(nx, ny, nz, 1, seed=42, lo=-5, hi=5)
    halo = out.copy()
    oracle.do_ordered(space, "PREFIX", r, 1, out, 1)
    ri = np.moveaxis(oracle.interior(r, 1), axis, -1)
    h_last = np.moveaxis(halo, axis, -1)  # ordered axis last
    before = h_last[1:-1, 1:-1, 0] if inc else h_last[1:-1, 1:-1, -1]
    seq = ri if inc else ri[..., ::-1]
    cs = np.cumsum(np.concatenate([before[..., None], seq], axis=-1), axis=-1)[..., 1:]
    cs = cs if inc else cs[..., ::-1]
    assert np.array_equal(np.moveaxis(oracle.interior(out, 1), axis, -1), cs)


def test_ordered_diamond_pascal_binomials(og):
    # Pascal's recurrence with 1s on the boundary gives C(i+j, i)
    n = 24
    out = oracle.alloc(n, n, 2, 1)
    out[:, 0, :] = 1.0
    out[:, :, 0] = 1.0
    oracle.do_ordered("DIAMOND", "PASCAL", None, 0, out, 1)
    for z in (1, 2):
        for y in range(n):
            for x in range(n):
                assert out[z, y + 1, x + 1] == math.comb(x + y + 2, x + 1)


@pytest.mark.parametrize("op", ["JACOBI7", "VARCOEF8"])
def test_dependency_cone_windows(og, op):
    # The full-size GPU tests compare windows of a jacobi_run too large for the
    # oracle: each window is grown by one point per sweep per side (clipped at
    # the physical boundary) and run alone.  Check that reading on a size the
    # oracle runs whole: the cone windows equal the whole-domain result.
    N, w, iters, check, seed = 36, 6, 5, 2, 99
    nc = 7 if op == "VARCOEF8" else 0
    u = oracle.alloc(N, N, N, 1)
    oracle.fill_random(u, 1, seed, 0)
    cs = [oracle.fill_random(oracle.alloc(N, N, N, 0), 0, seed, 2 + i, 0.125) for i in range(nc)]
    full, _ = oracle.jacobi_run(op, u, oracle.alloc(N, N, N, 1), 1, iters, check, coeffs=cs or None, ch=0)
    full = oracle.interior(full, 1)
    for o in [(0, 0, 0), (N - w, N - w, N - w), (14, 3, 29), (11, 17, 13)]:
        lo = [max(0, c - iters) for c in o]
        hi = [min(N, c + w + iters) for c in o]
        b = [hi[k] - lo[k] for k in range(3)]
        ua = oracle.fill_random_window(oracle.alloc(*b, 1), 1, lo, (N, N, N), seed, 0)
        ca = [oracle.fill_random_window(oracle.alloc(*b, 0), 0, lo, (N, N, N), seed, 2 + i, 0.125)
              for i in range(nc)]
        fin, _ = oracle.jacobi_run(op, ua, oracle.alloc(*b, 1), 1, iters, check, coeffs=ca or None, ch=0)
        d = [o[k] - lo[k] for k in range(3)]
        got = oracle.interior(fin, 1)[d[2]:d[2] + w, d[1]:d[1] + w, d[0]:d[0] + w]
        want = full[o[2]:o[2] + w, o[1]:o[1] + w, o[0]:o[0] + w]
        assert np.array_equal(got, want), o
    # the window's own halo holds the exact initial values, so growing by
    # iters - 1 is the tight bound: iters - 2 must differ (the check has teeth)
    if op == "JACOBI7":
        o = (15, 15, 15)
        lo = [c - iters + 2 for c in o]
        b = [w + 2 * (iters - 2)] * 3
        ua = oracle.fill_random_window(oracle.alloc(*b, 1), 1, lo, (N, N, N), seed, 0)
        fin, _ = oracle.jacobi_run(op, ua, oracle.alloc(*b, 1), 1, iters, check, ch=0)
        k = iters - 2
        got = oracle.interior(fin, 1)[k:k + w, k:k + w, k:k + w]
        assert not np.array_equal(got, full[15:15 + w, 15:15 + w, 15:15 + w])
