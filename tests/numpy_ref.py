"""Brute-force numpy evaluation of the catalogue trees on tiny grids.

An independent second implementation (whole-array shifted views instead of the
oracle's per-point accessor loops) used ONLY to cross-check the C++ oracle's
indexing and layout on small inputs.  Trees: DESIGN.md §3 (R1-R8).
"""
from __future__ import annotations

import numpy as np


def _sh(u, h, dx, dy, dz):
    """View of u shifted by (dx,dy,dz) over the interior (u has halo h)."""
    nz, ny, nx = (s - 2 * h for s in u.shape)
    return u[h + dz:h + dz + nz, h + dy:h + dy + ny, h + dx:h + dx + nx]


def fig1b(u, h):
    T = u.dtype.type
    s = T(6) * _sh(u, h, 0, 0, 0)
    for d in [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]:
        s = s - _sh(u, h, *d)
    return (T(1) / T(36)) * s


def sum6(u, h):
    sx = _sh(u, h, -1, 0, 0) + _sh(u, h, 1, 0, 0)
    sy = _sh(u, h, 0, -1, 0) + _sh(u, h, 0, 1, 0)
    sz = _sh(u, h, 0, 0, -1) + _sh(u, h, 0, 0, 1)
    return (sx + sy) + sz


def lap7(u, h):
    T = u.dtype.type
    return sum6(u, h) - T(6) * _sh(u, h, 0, 0, 0)


def jacobi7(u, h):
    T = u.dtype.type
    return sum6(u, h) * (T(1) / T(6))


def bracket27(u, h):
    T = u.dtype.type
    C, X, D = {}, {}, {}
    for q in (-1, 0, 1):
        C[q] = _sh(u, h, 0, 0, q)
        X[q] = (_sh(u, h, -1, 0, q) + _sh(u, h, 1, 0, q)) + (_sh(u, h, 0, -1, q) + _sh(u, h, 0, 1, q))
        D[q] = (_sh(u, h, -1, -1, q) + _sh(u, h, 1, -1, q)) + (_sh(u, h, -1, 1, q) + _sh(u, h, 1, 1, q))
    Sf = X[0] + (C[-1] + C[1])
    Se = D[0] + (X[-1] + X[1])
    Sc = D[-1] + D[1]
    return (T(14) * Sf + T(3) * Se) + Sc


def lap27(u, h):
    T = u.dtype.type
    return (bracket27(u, h) - T(128) * _sh(u, h, 0, 0, 0)) / T(30)


def jacobi27(u, h):
    T = u.dtype.type
    return bracket27(u, h) * T(0.0078125)


def varcoef8(grids, halos):
    u, hu = grids[0], halos[0]
    c = [_sh(g, hh, 0, 0, 0) for g, hh in zip(grids[1:], halos[1:])]
    a = c[0] * _sh(u, hu, 0, 0, 0)
    for ci, d in zip(c[1:], [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]):
        a = a + ci * _sh(u, hu, *d)
    return a


def apply(op, grids, halos):
    if op == "VARCOEF8":
        return varcoef8(grids, halos)
    return {"FIG1B": fig1b, "LAP7": lap7, "JACOBI7": jacobi7, "LAP27": lap27,
            "JACOBI27": jacobi27}[op](grids[0], halos[0])
