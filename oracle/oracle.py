"""ctypes + numpy front end of the C++ oracle (TEST INFRASTRUCTURE ONLY).

Grids here are numpy arrays in the oracle's dense layout
``[(nz+2h), (ny+2h), (nx+2h)]`` (x fastest), float64 or float32.
Every function cites the oracle routine it calls; the arithmetic lives in
``gscl_oracle.cpp`` only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gscl_oracle.cpp")
_LIB = os.path.join(_HERE, "libgscl_oracle.so")

# The oracle's own numbering; the tests map these by NAME onto the ABI's.
OPS = {"FIG1B": 0, "LAP7": 1, "JACOBI7": 2, "LAP27": 3, "JACOBI27": 4, "VARCOEF8": 5}
ROPS = {"VALUE": 0, "SQ": 1, "ABSDIFF": 2, "CONV": 3, "RESID7_SQ": 4, "RESID27_SQ": 5,
        "JACOBI7_RESID7_SQ": 6, "JACOBI27_RESID27_SQ": 7, "FIG1B_CONV": 8}
COMBINES = {"SUM": 0, "MAX": 1, "MIN": 2, "AND": 3}
ARITY = {"FIG1B": 1, "LAP7": 1, "JACOBI7": 1, "LAP27": 1, "JACOBI27": 1, "VARCOEF8": 8}

__all__ = ["OPS", "ROPS", "COMBINES", "ARITY", "build", "lib", "splitmix64", "alloc",
           "fill_random", "fill_random_window", "digest", "do_all", "do_reduce", "jacobi_run", "num_threads",
           "set_threads", "interior", "converge_run", "rbgs_run", "do_ordered", "SPACES", "OOPS"]

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2, no FP contraction, no fast-math, OpenMP."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", tmp, _SRC]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, i32, u64, vp, dp = (ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p,
                                 ctypes.POINTER(ctypes.c_double))
        L.og_splitmix64.argtypes = [u64]
        L.og_splitmix64.restype = u64
        L.og_fill_random.argtypes = [i32, vp, i64, i64, i64, i32, i64, u64, ctypes.c_uint32,
                                     ctypes.c_double]
        L.og_fill_random_window.argtypes = [i32, vp, i64, i64, i64, i32, i64, i64, i64, i64, i64,
                                            i64, u64, ctypes.c_uint32, ctypes.c_double]
        L.og_digest.argtypes = [i32, vp, i64, i64, i64, i32, i64]
        L.og_digest.restype = u64
        L.og_do_all.argtypes = [i32, i32, ctypes.POINTER(vp), ctypes.POINTER(i32), i32, vp, i32,
                                i64, i64, i64, ctypes.POINTER(i64)]
        L.og_do_reduce.argtypes = [i32, i32, ctypes.POINTER(vp), ctypes.POINTER(i32), i32, vp,
                                   i32, i64, i64, i64, ctypes.POINTER(i64), i32, ctypes.c_double,
                                   dp, dp]
        L.og_jacobi_run.argtypes = [i32, i32, vp, vp, i32, ctypes.POINTER(vp), i32, i64, i64, i64,
                                    i32, i32, dp, ctypes.POINTER(i32)]
        L.og_converge_run.argtypes = [i32, i32, vp, vp, i32, i64, i64, i64, ctypes.c_double, i32,
                                      ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]
        L.og_rbgs_run.argtypes = [i32, vp, i32, i64, i64, i64, i64, i32, i32, dp]
        L.og_do_ordered.argtypes = [i32, i32, i32, vp, i32, vp, i32, i64, i64, i64]
        L.og_num_threads.restype = i32
        L.og_set_threads.argtypes = [i32]
        _lib = L
    return _lib


def num_threads() -> int:
    return lib().og_num_threads()


def set_threads(n: int) -> None:
    lib().og_set_threads(n)


def splitmix64(x: int) -> int:
    return lib().og_splitmix64(x & (2**64 - 1))


def _dt(a: np.ndarray) -> int:
    if a.dtype == np.float64:
        return 0
    if a.dtype == np.float32:
        return 1
    raise TypeError(a.dtype)


def _halo(a: np.ndarray, nx: int) -> int:
    h2 = a.shape[2] - nx
    assert h2 >= 0 and h2 % 2 == 0
    return h2 // 2


def alloc(nx: int, ny: int, nz: int, h: int, dtype=np.float64) -> np.ndarray:
    return np.zeros((nz + 2 * h, ny + 2 * h, nx + 2 * h), dtype=dtype)


def interior(a: np.ndarray, h: int) -> np.ndarray:
    return a[h:a.shape[0] - h, h:a.shape[1] - h, h:a.shape[2] - h]


def _dims(a: np.ndarray, h: int):
    return a.shape[2] - 2 * h, a.shape[1] - 2 * h, a.shape[0] - 2 * h


def fill_random(a: np.ndarray, h: int, seed: int, grid_id: int, scale: float = 1.0,
                z_off: int = 0) -> np.ndarray:
    """og_fill_random: reading R9 generator over global interior indices; zero halo."""
    assert a.flags.c_contiguous
    nx, ny, nz = _dims(a, h)
    lib().og_fill_random(_dt(a), a.ctypes.data, nx, ny, nz, h, z_off, seed, grid_id, scale)
    return a


def fill_random_window(a: np.ndarray, h: int, off, global_dims, seed: int, grid_id: int,
                       scale: float = 1.0) -> np.ndarray:
    """og_fill_random_window: the window of the global field whose interior
    origin is global point off = (x, y, z); outside the global interior -> 0."""
    bx, by, bz = _dims(a, h)
    NX, NY, NZ = global_dims
    lib().og_fill_random_window(_dt(a), a.ctypes.data, bx, by, bz, h, off[0], off[1], off[2],
                                NX, NY, NZ, seed, grid_id, scale)
    return a


def digest(a: np.ndarray, h: int, z_off: int = 0) -> int:
    """og_digest: order-independent 64-bit interior digest (reading R10)."""
    assert a.flags.c_contiguous
    nx, ny, nz = _dims(a, h)
    return lib().og_digest(_dt(a), a.ctypes.data, nx, ny, nz, h, z_off)


def _ptrs(arrs):
    return (ctypes.c_void_p * len(arrs))(*[x.ctypes.data for x in arrs])


def _rng(rng, nx, ny, nz):
    if rng is None:
        rng = (0, nx, 0, ny, 0, nz)
    return (ctypes.c_int64 * 6)(*rng)


def do_all(op: str, ins, halos, out: np.ndarray, out_h: int, rng=None) -> None:
    """og_do_all: out(p) = OP(ins)(p) for p in the local range (default: all interior)."""
    nx, ny, nz = _dims(out, out_h)
    for a in list(ins) + [out]:
        assert a.flags.c_contiguous and a.dtype == out.dtype
    rc = lib().og_do_all(OPS[op], _dt(out), _ptrs(ins), (ctypes.c_int * len(halos))(*halos),
                         len(ins), out.ctypes.data, out_h, nx, ny, nz, _rng(rng, nx, ny, nz))
    if rc != 0:
        raise ValueError(f"og_do_all({op}) rejected its arguments")


def do_reduce(rop: str, grids, halos, combine: str, rng=None, eps: float = 0.0,
              out: np.ndarray | None = None, out_h: int = 0, dims=None):
    """og_do_reduce -> (result, sum |val|).  Fused rops also write ``out``."""
    g0 = grids[0]
    nx, ny, nz = dims if dims is not None else _dims(g0, halos[0])
    r = ctypes.c_double()
    a = ctypes.c_double()
    rc = lib().og_do_reduce(ROPS[rop], _dt(g0), _ptrs(grids), (ctypes.c_int * len(halos))(*halos),
                            len(grids), None if out is None else out.ctypes.data, out_h, nx, ny,
                            nz, _rng(rng, nx, ny, nz), COMBINES[combine], eps, ctypes.byref(r),
                            ctypes.byref(a))
    if rc != 0:
        raise ValueError(f"og_do_reduce({rop}) rejected its arguments")
    return r.value, a.value


def jacobi_run(op: str, u: np.ndarray, v: np.ndarray, h: int, iters: int, check_every: int,
               coeffs=None, ch: int = 0):
    """og_jacobi_run -> (final_iterate_array, history list).  u and v are updated in place."""
    nx, ny, nz = _dims(u, h)
    nhist = iters // check_every + 1 if check_every > 0 else 0
    hist = (ctypes.c_double * max(nhist, 1))()
    fin = ctypes.c_int()
    cs = coeffs or []
    rc = lib().og_jacobi_run(OPS[op], _dt(u), u.ctypes.data, v.ctypes.data, h,
                             _ptrs(cs) if cs else None, ch, nx, ny, nz, iters, check_every, hist,
                             ctypes.byref(fin))
    if rc != 0:
        raise ValueError(f"og_jacobi_run({op}) rejected its arguments")
    return (u if fin.value == 0 else v), [hist[i] for i in range(nhist)]


def converge_run(op: str, u: np.ndarray, v: np.ndarray, h: int, eps: float, max_iters: int):
    """og_converge_run -> (final_iterate, iterations, converged)."""
    nx, ny, nz = _dims(u, h)
    it, conv, fin = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rc = lib().og_converge_run(OPS[op], _dt(u), u.ctypes.data, v.ctypes.data, h, nx, ny, nz, eps,
                               max_iters, ctypes.byref(it), ctypes.byref(conv), ctypes.byref(fin))
    if rc != 0:
        raise ValueError(f"og_converge_run({op}) rejected its arguments")
    return (u if fin.value == 0 else v), it.value, bool(conv.value)


def rbgs_run(u: np.ndarray, h: int, iters: int, check_every: int, z_off: int = 0):
    """og_rbgs_run: red-black Gauss-Seidel (NEXT-3), u updated in place -> history."""
    nx, ny, nz = _dims(u, h)
    nhist = iters // check_every + 1 if check_every > 0 else 0
    hist = (ctypes.c_double * max(nhist, 1))()
    rc = lib().og_rbgs_run(_dt(u), u.ctypes.data, h, nx, ny, nz, z_off, iters, check_every, hist)
    if rc != 0:
        raise ValueError("og_rbgs_run rejected its arguments")
    return [hist[i] for i in range(nhist)]


SPACES = {"I_INC": 0, "I_DEC": 1, "J_INC": 2, "J_DEC": 3, "K_INC": 4, "K_DEC": 5, "DIAMOND": 6}
OOPS = {"PREFIX": 0, "PASCAL": 1}


def do_ordered(space: str, op: str, inp, in_h: int, out: np.ndarray, out_h: int) -> None:
    """og_do_ordered (NEXT-4): literal ordered evaluation."""
    nx, ny, nz = _dims(out, out_h)
    rc = lib().og_do_ordered(SPACES[space], OOPS[op], _dt(out), None if inp is None else inp.ctypes.data,
                             in_h, out.ctypes.data, out_h, nx, ny, nz)
    if rc != 0:
        raise ValueError("og_do_ordered rejected its arguments")
