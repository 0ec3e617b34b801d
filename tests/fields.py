"""Seeded / analytic INPUT fields for the tests (no stencil arithmetic here).

Both the oracle and the GPU path receive the same arrays (the GPU via
``copy_from_host``).  All arrays use the oracle's dense layout
``[(nz+2h), (ny+2h), (nx+2h)]`` with interior coordinate x = 0..nx-1 at
array index x+h.
"""
from __future__ import annotations

import math

import numpy as np


def coords(nx, ny, nz, h):
    """Interior-coordinate arrays X, Y, Z over the WHOLE padded array (halo cells
    get coordinates -h.. and n..n+h-1), shape (nz+2h, ny+2h, nx+2h)."""
    z = np.arange(-h, nz + h, dtype=np.float64)[:, None, None]
    y = np.arange(-h, ny + h, dtype=np.float64)[None, :, None]
    x = np.arange(-h, nx + h, dtype=np.float64)[None, None, :]
    return np.broadcast_arrays(x, y, z)


def quadratic(nx, ny, nz, h, c, dtype=np.float64):
    """Integer quadratic  a x^2 + b y^2 + c z^2 + d xy + e yz + f xz + g x + hh y + k z + l
    evaluated at every cell INCLUDING the halo (so the halo carries the field's own
    boundary values).  c = (a, b, c, d, e, f, g, hh, k, l), small integers."""
    X, Y, Z = coords(nx, ny, nz, h)
    a, b, cc, d, e, f, g, hh, k, l = c
    v = a * X * X + b * Y * Y + cc * Z * Z + d * X * Y + e * Y * Z + f * X * Z + g * X + hh * Y + k * Z + l
    return np.ascontiguousarray(v.astype(dtype))


def sine_mode(n, h, dtype=np.float64):
    """Lowest Dirichlet eigenmode on an n^3 interior with zero halo:
    U = sin(t(x+1)) sin(t(y+1)) sin(t(z+1)), t = pi/(n+1)."""
    t = math.pi / (n + 1)
    s = np.sin(t * (np.arange(n) + 1.0))
    a = np.zeros((n + 2 * h,) * 3, dtype=dtype)
    a[h:n + h, h:n + h, h:n + h] = (s[:, None, None] * s[None, :, None] * s[None, None, :]).astype(dtype)
    return a


def spike(n, h, value, dtype=np.float64):
    """n^3 interior (n odd), zero everywhere except `value` at the centre."""
    a = np.zeros((n + 2 * h,) * 3, dtype=dtype)
    c = n // 2 + h
    a[c, c, c] = value
    return a


def constant(nx, ny, nz, h, value, dtype=np.float64, halo_too=True):
    a = np.zeros((nz + 2 * h, ny + 2 * h, nx + 2 * h), dtype=dtype)
    if halo_too:
        a[...] = value
    else:
        a[h:nz + h, h:ny + h, h:nx + h] = value
    return a


def seeded_uniform(nx, ny, nz, h, seed, dtype=np.float64, lo=0.0, hi=1.0):
    """numpy-PCG64 uniform interior with zero halo (a second, non-splitmix input family)."""
    rng = np.random.default_rng(seed)
    a = np.zeros((nz + 2 * h, ny + 2 * h, nx + 2 * h), dtype=dtype)
    a[h:nz + h, h:ny + h, h:nx + h] = rng.uniform(lo, hi, size=(nz, ny, nx)).astype(dtype)
    return a
