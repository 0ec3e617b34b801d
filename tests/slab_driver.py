"""Slab-mode oracle driver (test infrastructure): the oracle run as P z-slabs
with explicit halo-plane copies, the CPU model of the multi-GPU path
("tiled == monolithic").

Split rule (R13): the first nz mod P slabs get
ceil(nz/P) planes, the rest floor(nz/P).
"""
from __future__ import annotations

import numpy as np

import oracle


def slab_bounds(nz: int, P: int):
    base, rem = divmod(nz, P)
    out, z = [], 0
    for r in range(P):
        n = base + (1 if r < rem else 0)
        out.append((z, z + n))
        z += n
    return out


def split(full: np.ndarray, h: int, P: int):
    """Cut a dense single-domain array into P slab arrays (each with its own
    halo planes, copied from the full array)."""
    nz = full.shape[0] - 2 * h
    return [np.ascontiguousarray(full[z0:z1 + 2 * h]) for (z0, z1) in slab_bounds(nz, P)]


def join(slabs, h: int) -> np.ndarray:
    parts = [s[h:s.shape[0] - h] for s in slabs]
    lo = slabs[0][:h]
    hi = slabs[-1][slabs[-1].shape[0] - h:]
    return np.ascontiguousarray(np.concatenate([lo] + parts + [hi], axis=0))


def exchange(slabs, h: int) -> None:
    """Ghost planes := neighbour's boundary interior planes.
    Physical-boundary halo planes (rank 0 bottom, rank P-1 top) are untouched."""
    for r in range(len(slabs) - 1):
        lo, hi = slabs[r], slabs[r + 1]
        nlo = lo.shape[0] - 2 * h
        # top ghost planes of r  <- first interior planes of r+1
        lo[nlo + h:nlo + 2 * h] = hi[h:2 * h]
        # bottom ghost planes of r+1 <- last interior planes of r
        hi[0:h] = lo[nlo:nlo + h]


def jacobi_slabs(op: str, u_full: np.ndarray, h: int, P: int, iters: int):
    """JACOBI7 / JACOBI27 for `iters` sweeps as P slabs; returns the joined result."""
    us = split(u_full, h, P)
    vs = [s.copy() for s in us]  # v carries the same (physical) halo shell
    for _ in range(iters):
        exchange(us, h)
        for a, b in zip(us, vs):
            oracle.do_all(op, [a], [h], b, h)
        us, vs = vs, us
    return join(us, h)
