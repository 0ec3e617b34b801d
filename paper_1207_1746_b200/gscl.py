"""Thin ctypes binding of the C ABI in include/gscl.h (argument marshalling only).

Every computation runs in libgscl.so's kernels.  PyTorch supplies the device
memory (grids are torch uint8 buffers wrapped with gscl_grid_wrap), the CUDA
stream (torch's current stream at init) and, on multi-rank runs, the process
group used to broadcast the NCCL unique id.  There is no CPU fallback: if the
shared library is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GSCL_LIB selects another build of the same ABI (the ablation build,
# libgscl_ablations.so — see build.py); the default is the product library.
LIB_PATH = os.environ.get("GSCL_LIB") or os.path.join(_HERE, "libgscl.so")

# ---- enums (values mirror include/gscl.h) ------------------------------------
F64, F32 = 0, 1
OK = 0
STATUS = {0: "GSCL_OK", 1: "GSCL_E_INVALID_ARG", 2: "GSCL_E_INVALID_DOMAIN",
          3: "GSCL_E_SHAPE_MISMATCH", 4: "GSCL_E_HALO_VIOLATION", 5: "GSCL_E_ARITY",
          6: "GSCL_E_RANGE", 7: "GSCL_E_DTYPE", 8: "GSCL_E_STATE", 9: "GSCL_E_OOM",
          10: "GSCL_E_CUDA", 11: "GSCL_E_NCCL", 12: "GSCL_E_UNSUPPORTED",
          13: "GSCL_E_TIMEOUT"}
OPS = {"FIG1B": 0, "LAP7": 1, "JACOBI7": 2, "LAP27": 3, "JACOBI27": 4, "VARCOEF8": 5}
ROPS = {"VALUE": 0, "SQ": 1, "ABSDIFF": 2, "CONV": 3, "RESID7_SQ": 4, "RESID27_SQ": 5,
        "JACOBI7_RESID7_SQ": 6, "JACOBI27_RESID27_SQ": 7, "FIG1B_CONV": 8}
COMBINES = {"SUM": 0, "MAX": 1, "MIN": 2, "AND": 3}
SPACES = {"I_INC": 0, "I_DEC": 1, "J_INC": 2, "J_DEC": 3, "K_INC": 4, "K_DEC": 5, "DIAMOND": 6}
OOPS = {"PREFIX": 0, "PASCAL": 1}


class GsclError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Range(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("x0", "x1", "y0", "y1", "z0", "z1")]


class HaloOp(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int), ("is_send", ctypes.c_int), ("offset", ctypes.c_int64),
                ("bytes", ctypes.c_int64)]


class PassPeer(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_void_p * 2), ("hi", ctypes.c_void_p * 2), ("lo_flag", ctypes.c_void_p),
                ("hi_flag", ctypes.c_void_p)]


class PassXfer(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int), ("is_send", ctypes.c_int), ("z", ctypes.c_int64),
                ("ghost_plane", ctypes.c_int)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1207_1746_b200.build` "
                          "(the CUDA library is required; there is no fallback)")
    L = ctypes.CDLL(LIB_PATH)
    i32, i64, u64, vp, sz = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t
    G = ctypes.c_void_p
    P = ctypes.POINTER
    sig = {
        "gscl_get_nccl_unique_id": [vp],
        "gscl_init": [i32, i32, vp, i32, vp],
        "gscl_finalize": [],
        "gscl_sync": [],
        "gscl_grid_create": [i64, i64, i64, i32, i32, P(G)],
        "gscl_grid_wrap": [vp, sz, i64, i64, i64, i32, i32, P(G)],
        "gscl_grid_destroy": [G],
        "gscl_grid_bytes": [i64, i64, i64, i32, i32, i32, i32, P(sz)],
        "gscl_grid_layout": [G, P(i64), P(i64), P(i64), P(i64)],
        "gscl_grid_device_ptr": [G, P(vp)],
        "gscl_slab_range": [i64, i32, i32, P(i64), P(i64)],
        "gscl_grid_fill_random": [G, u64, ctypes.c_uint32, ctypes.c_double],
        "gscl_grid_fill_const": [G, ctypes.c_double],
        "gscl_grid_copy_to_host": [G, vp, sz],
        "gscl_grid_copy_from_host": [G, vp, sz],
        "gscl_grid_copy_from_host_async": [G, vp, sz],
        "gscl_grid_copy_to_host_async": [G, vp, sz],
        "gscl_grid_digest": [G, P(u64)],
        "gscl_swap": [G, G],
        "gscl_do_all": [i32, P(G), i32, G, P(Range), P(ctypes.c_double), i32],
        "gscl_do_reduce": [i32, P(G), i32, G, i32, P(Range), P(ctypes.c_double), i32,
                           P(ctypes.c_double)],
        "gscl_halo_exchange": [P(G), i32],
        "gscl_halo_exchange_depth": [P(G), i32, i32],
        "gscl_halo_plan": [i64, i64, i64, i32, i32, i32, i32, P(HaloOp), P(i32)],
        "gscl_pass_plan": [i64, i64, i64, i32, i32, i32, i32, P(PassXfer), P(i32)],
        "gscl_do_all_pass2": [i32, G, G, vp, i32, i32, P(PassPeer)],
        "gscl_do_all_pass2_coeffs": [i32, G, P(G), i32, G, vp, vp, i32, i32, P(PassPeer)],
        "gscl_pass_units": [i64, i64, i32, P(i64)],
        "gscl_pass_units_op": [i32, i64, i64, i32, P(i64)],
        "gscl_peer_export": [G, G, vp, sz, P(sz)],
        "gscl_peer_import": [G, G, vp, sz],
        "gscl_jacobi_run": [i32, G, G, P(G), i32, i32, i32, P(ctypes.c_double)],
        "gscl_converge_run": [i32, G, G, ctypes.c_double, i32, i32, P(i32), P(i32)],
        "gscl_rbgs_run": [G, i32, i32, P(ctypes.c_double)],
        "gscl_do_ordered": [i32, i32, G, G],
        "gscl_timing_enable": [i32],
        "gscl_timing_read": [P(ctypes.c_double), P(i64), P(i64)],
        "gscl_set_option": [ctypes.c_char_p, i64],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = i32
    L.gscl_last_error.restype = ctypes.c_char_p
    L.gscl_last_error.argtypes = []
    L.gscl_version.restype = ctypes.c_char_p
    L.gscl_version.argtypes = []
    return L


lib = _load()


def _ck(status: int) -> None:
    if status != OK:
        raise GsclError(status, lib.gscl_last_error().decode())


def version() -> str:
    return lib.gscl_version().decode()


def slab_range(nz: int, rank: int, world: int):
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _ck(lib.gscl_slab_range(nz, rank, world, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def grid_bytes(nx, ny, nz, halo, dtype=F64, rank=0, world=1) -> int:
    n = ctypes.c_size_t()
    _ck(lib.gscl_grid_bytes(nx, ny, nz, halo, dtype, rank, world, ctypes.byref(n)))
    return n.value


def halo_plan(nx, ny, nz, halo, dtype=F64, rank=0, world=1):
    """The exchange ops of `rank`: [(peer, is_send, byte_offset, bytes)]."""
    ops = (HaloOp * 4)()
    n = ctypes.c_int()
    _ck(lib.gscl_halo_plan(nx, ny, nz, halo, dtype, rank, world, ops, ctypes.byref(n)))
    return [(ops[i].peer, ops[i].is_send, ops[i].offset, ops[i].bytes) for i in range(n.value)]


def pass_plan(nx, ny, nz, halo, dtype=F64, rank=0, world=1):
    """The depth-2 exchange of a two-sweep pass: [(peer, is_send, z, ghost_plane)]
    (z local; ghost_plane 0 = in the grid, 1 / 2 = ghost buffer plane 0 / 1)."""
    ops = (PassXfer * 8)()
    n = ctypes.c_int()
    _ck(lib.gscl_pass_plan(nx, ny, nz, halo, dtype, rank, world, ops, ctypes.byref(n)))
    return [(ops[i].peer, ops[i].is_send, ops[i].z, ops[i].ghost_plane) for i in range(n.value)]


def do_all_pass2(op: str, inp: "Grid", out: "Grid", ghost=None, phys_lo: bool = True,
                 phys_hi: bool = True, peer: Optional[dict] = None, coeffs: Sequence["Grid"] = (),
                 cghost=None) -> None:
    """One two-sweep pass of a slab whose z neighbours' planes the caller supplies
    (in's halo planes + `ghost`, a device tensor of 2 planes, when halo is 1).
    peer: {"lo": [ptr, ptr], "hi": [ptr, ptr], "lo_flag": ptr, "hi_flag": ptr}
    (device addresses, None = skip) — the pass also stores its boundary planes
    there and bumps the flags (the peer-memory halo transport)."""
    ptr = ghost.data_ptr() if ghost is not None else None
    pp = None
    if peer is not None:
        pp = PassPeer()
        for i in range(2):
            pp.lo[i] = peer.get("lo", [None, None])[i]
            pp.hi[i] = peer.get("hi", [None, None])[i]
        pp.lo_flag = peer.get("lo_flag")
        pp.hi_flag = peer.get("hi_flag")
        pp = ctypes.byref(pp)
    if coeffs or op != "JACOBI7":
        cptr = cghost.data_ptr() if cghost is not None else None
        _ck(lib.gscl_do_all_pass2_coeffs(OPS[op], inp.handle, _handles(coeffs) if coeffs else None, len(coeffs),
                                         out.handle, ptr, cptr, int(phys_lo), int(phys_hi), pp))
        return
    _ck(lib.gscl_do_all_pass2(OPS[op], inp.handle, out.handle, ptr, int(phys_lo), int(phys_hi), pp))


def peer_export(u: "Grid", v: "Grid") -> bytes:
    """This rank's IPC blob for the peer-memory transport (see peer_setup)."""
    n = ctypes.c_size_t()
    _ck(lib.gscl_peer_export(u.handle, v.handle, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _ck(lib.gscl_peer_export(u.handle, v.handle, buf, n.value, ctypes.byref(n)))
    return buf.raw[: n.value]


def peer_import(u: "Grid", v: "Grid", blobs: Sequence[bytes]) -> None:
    each = len(blobs[0])
    assert all(len(b) == each for b in blobs)
    arr = ctypes.create_string_buffer(b"".join(blobs), each * len(blobs))
    _ck(lib.gscl_peer_import(u.handle, v.handle, arr, each))


def peer_setup(u: "Grid", v: "Grid", all_gather) -> None:
    """Collective: export, all-gather the blobs in rank order with
    `all_gather(bytes) -> list[bytes]` (e.g. over torch.distributed), import,
    and switch jacobi_run to the peer-memory transport."""
    blobs = all_gather(peer_export(u, v))
    peer_import(u, v, blobs)
    set_option("transport", 1)


def pass_units(nx: int, ny: int, dtype: int = F64, op: str = "JACOBI7") -> int:
    n = ctypes.c_int64()
    _ck(lib.gscl_pass_units_op(OPS[op], nx, ny, dtype, ctypes.byref(n)))
    return n.value


def layout_of(nx, ny, nz, halo, dtype=F64, rank=0, world=1):
    """Host-side layout numbers of a slab (no GPU): pitch, z range, origin offset."""
    es = 8 if dtype == F64 else 4
    ox = 128 // es
    pitch = (ox + nx + halo + ox - 1) // ox * ox
    z0, z1 = slab_range(nz, rank, world)
    return {"pitch": pitch, "rows": ny + 2 * halo, "planes": (z1 - z0) + 2 * halo, "ox": ox,
            "z_begin": z0, "z_end": z1, "es": es,
            "bytes": grid_bytes(nx, ny, nz, halo, dtype, rank, world)}


def get_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _ck(lib.gscl_get_nccl_unique_id(buf))
    return buf.raw


_state = {"inited": False, "rank": 0, "world": 1}


def init(rank: int = 0, world: int = 1, device: int = 0, stream=None, nccl_id: Optional[bytes] = None,
         process_group=None, use_nccl: bool = True) -> None:
    """gscl_init on torch's current stream of `device`.  For world > 1 the NCCL
    unique id is created on rank 0 and broadcast with torch.distributed
    (use_nccl=False: no communicator — only the peer-memory transport)."""
    import torch
    torch.cuda.set_device(device)
    if world > 1 and nccl_id is None and use_nccl:
        import torch.distributed as dist
        t = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            t[:] = torch.frombuffer(bytearray(get_nccl_unique_id()), dtype=torch.uint8)
        dist.broadcast(t, src=0, group=process_group)
        nccl_id = bytes(t.numpy().tobytes())
    if stream is None:
        cur = torch.cuda.current_stream(device)
        if cur.cuda_stream == 0:
            # give the library (and torch on this thread) a dedicated stream so
            # grid allocations, fills and library kernels are ordered together
            cur = torch.cuda.Stream(device)
            torch.cuda.set_stream(cur)
        _state["stream"] = cur
        stream = cur.cuda_stream
    idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    _ck(lib.gscl_init(rank, world, idbuf, device, ctypes.c_void_p(stream)))
    _state.update(inited=True, rank=rank, world=world)


def finalize() -> None:
    _ck(lib.gscl_finalize())
    _state["inited"] = False


def sync() -> None:
    _ck(lib.gscl_sync())


def set_option(name: str, value: int) -> None:
    _ck(lib.gscl_set_option(name.encode(), value))


def has_ablations() -> bool:
    """True when the loaded library is the ablation build (libgscl_ablations.so,
    build.py --ablations): its extra knobs (sweep_impl, variant, zchunks, sched,
    stages, l2promo, zalt) are accepted; the product library rejects them."""
    st = lib.gscl_set_option(b"sweep_impl", 1)
    if st == OK:
        lib.gscl_set_option(b"sweep_impl", 0)
        return True
    return False


def timing_enable(on: bool = True) -> None:
    _ck(lib.gscl_timing_enable(1 if on else 0))


def timing_read():
    """-> (ms[4], n[4], launches): per sweep kind (0 do_all, 1 fused, 2 reduce-only, 3 two-sweep)
    the summed device ms and launch counts, and all kernels launched."""
    ms = (ctypes.c_double * 4)()
    n = (ctypes.c_int64 * 4)()
    k = ctypes.c_int64()
    _ck(lib.gscl_timing_read(ms, n, ctypes.byref(k)))
    return list(ms), list(n), k.value


class Grid:
    """A grid whose HBM storage is a torch buffer wrapped by gscl_grid_wrap."""

    def __init__(self, nx: int, ny: int, nz: int, halo: int = 1, dtype: int = F64, device=None):
        import torch
        self.nx, self.ny, self.nz, self.halo, self.dtype = nx, ny, nz, halo, dtype
        self.nbytes = grid_bytes(nx, ny, nz, halo, dtype, _state["rank"], _state["world"])
        dev = device if device is not None else torch.cuda.current_device()
        self._buf = torch.zeros(self.nbytes, dtype=torch.uint8, device=f"cuda:{dev}")
        h = ctypes.c_void_p()
        _ck(lib.gscl_grid_wrap(ctypes.c_void_p(self._buf.data_ptr()), self.nbytes, nx, ny, nz, halo,
                               dtype, ctypes.byref(h)))
        self.handle = h
        p, z0, z1, off = (ctypes.c_int64() for _ in range(4))
        _ck(lib.gscl_grid_layout(h, ctypes.byref(p), ctypes.byref(z0), ctypes.byref(z1), ctypes.byref(off)))
        self.pitch, self.z_begin, self.z_end, self.origin_offset = p.value, z0.value, z1.value, off.value
        self.nzl = self.z_end - self.z_begin

    # storage bookkeeping: the C side may exchange storage between handles
    def _base(self) -> int:
        p = ctypes.c_void_p()
        _ck(lib.gscl_grid_device_ptr(self.handle, ctypes.byref(p)))
        return p.value or 0

    def destroy(self) -> None:
        if self.handle is not None:
            _ck(lib.gscl_grid_destroy(self.handle))
            self.handle = None
            self._buf = None

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == F64 else np.float32

    def dense_shape(self):
        h = self.halo
        return (self.nzl + 2 * h, self.ny + 2 * h, self.nx + 2 * h)

    def fill_random(self, seed: int, grid_id: int, scale: float = 1.0) -> "Grid":
        _ck(lib.gscl_grid_fill_random(self.handle, seed, grid_id, scale))
        return self

    def fill_const(self, value: float) -> "Grid":
        _ck(lib.gscl_grid_fill_const(self.handle, value))
        return self

    def to_host(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        a = out if out is not None else np.empty(self.dense_shape(), dtype=self.np_dtype)
        assert a.flags.c_contiguous and a.dtype == self.np_dtype and a.shape == self.dense_shape()
        _ck(lib.gscl_grid_copy_to_host(self.handle, ctypes.c_void_p(a.ctypes.data), a.nbytes))
        return a

    def from_host(self, a: np.ndarray) -> "Grid":
        a = np.ascontiguousarray(a, dtype=self.np_dtype)
        assert a.shape == self.dense_shape(), (a.shape, self.dense_shape())
        _ck(lib.gscl_grid_copy_from_host(self.handle, ctypes.c_void_p(a.ctypes.data), a.nbytes))
        return self

    def from_host_async(self, a: np.ndarray) -> "Grid":
        """gscl_grid_copy_from_host_async: returns at once; `a` is kept alive here
        until the next upload into this grid (keep it unmodified until used)."""
        assert a.flags.c_contiguous and a.dtype == self.np_dtype and a.shape == self.dense_shape()
        _ck(lib.gscl_grid_copy_from_host_async(self.handle, ctypes.c_void_p(a.ctypes.data), a.nbytes))
        self._pending_host = a
        return self

    def to_host_async(self, out: np.ndarray) -> np.ndarray:
        """gscl_grid_copy_to_host_async: returns at once; `out` holds the data
        after the next gscl.sync() (it is kept alive here until then)."""
        assert out.flags.c_contiguous and out.dtype == self.np_dtype and out.shape == self.dense_shape()
        _ck(lib.gscl_grid_copy_to_host_async(self.handle, ctypes.c_void_p(out.ctypes.data), out.nbytes))
        self._pending_out = out
        return out

    def digest(self) -> int:
        d = ctypes.c_uint64()
        _ck(lib.gscl_grid_digest(self.handle, ctypes.byref(d)))
        return d.value

    def device_view(self):
        """torch view of the padded local array, shape (planes, rows, pitch)."""
        import torch
        t = self._buf.view(torch.float64 if self.dtype == F64 else torch.float32)
        h = self.halo
        return t[: (self.nzl + 2 * h) * (self.ny + 2 * h) * self.pitch].view(
            self.nzl + 2 * h, self.ny + 2 * h, self.pitch)


def grid_create(nx, ny, nz, halo=1, dtype=F64) -> Grid:
    return Grid(nx, ny, nz, halo, dtype)


def _handles(grids: Sequence[Grid]):
    return (ctypes.c_void_p * max(len(grids), 1))(*[g.handle for g in grids])


def _range(r):
    if r is None:
        return None
    return ctypes.byref(Range(*[int(v) for v in r]))


def _swap_bufs(a: Grid, b: Grid) -> None:
    a._buf, b._buf = b._buf, a._buf


def swap(a: Grid, b: Grid) -> None:
    _ck(lib.gscl_swap(a.handle, b.handle))
    _swap_bufs(a, b)


def do_all(op: str, ins: Sequence[Grid], out: Grid, rng=None) -> None:
    _ck(lib.gscl_do_all(OPS[op], _handles(ins), len(ins), out.handle, _range(rng), None, 0))


def do_reduce(rop: str, grids: Sequence[Grid], combine: str = "SUM", out: Optional[Grid] = None,
              rng=None, eps: Optional[float] = None) -> float:
    res = ctypes.c_double()
    params = (ctypes.c_double * 1)(eps) if eps is not None else None
    _ck(lib.gscl_do_reduce(ROPS[rop], _handles(grids), len(grids), out.handle if out else None,
                           COMBINES[combine], _range(rng), params, 1 if eps is not None else 0,
                           ctypes.byref(res)))
    return res.value


def halo_exchange(grids: Sequence[Grid]) -> None:
    _ck(lib.gscl_halo_exchange(_handles(grids), len(grids)))


def halo_exchange_depth(grids: Sequence[Grid], depth: int) -> None:
    """gscl_halo_exchange_depth: depth 1 (h planes) or 2 (the two-sweep pass's
    exchange) over the current transport option (NCCL, or peer memory)."""
    _ck(lib.gscl_halo_exchange_depth(_handles(grids), len(grids), depth))


def jacobi_run(op: str, u: Grid, v: Grid, iters: int, check_every: int = 0,
               coeffs: Sequence[Grid] = ()) -> list:
    nh = iters // check_every + 1 if check_every > 0 else 0
    hist = (ctypes.c_double * max(nh, 1))()
    ub = u._base()
    _ck(lib.gscl_jacobi_run(OPS[op], u.handle, v.handle, _handles(coeffs) if coeffs else None,
                            len(coeffs), iters, check_every, hist if nh else None))
    if u._base() != ub:  # the library moved the final iterate's storage into u
        _swap_bufs(u, v)
    return [hist[i] for i in range(nh)]


def converge_run(op: str, u: Grid, v: Grid, eps: float, max_iters: int, batch: int = 16):
    """The paper's convergence loop -> (iterations, converged)."""
    it, conv = ctypes.c_int(), ctypes.c_int()
    ub = u._base()
    _ck(lib.gscl_converge_run(OPS[op], u.handle, v.handle, eps, max_iters, batch, ctypes.byref(it),
                              ctypes.byref(conv)))
    if u._base() != ub:
        _swap_bufs(u, v)
    return it.value, bool(conv.value)


def rbgs_run(u: Grid, iters: int, check_every: int = 0) -> list:
    """Red-black Gauss-Seidel (NEXT-3), in place on u -> residual history."""
    nh = iters // check_every + 1 if check_every > 0 else 0
    hist = (ctypes.c_double * max(nh, 1))()
    _ck(lib.gscl_rbgs_run(u.handle, iters, check_every, hist if nh else None))
    return [hist[i] for i in range(nh)]


def do_ordered(space: str, op: str, inp: Optional[Grid], out: Grid) -> None:
    """Ordered iteration spaces (NEXT-4)."""
    _ck(lib.gscl_do_ordered(SPACES[space], OOPS[op], inp.handle if inp is not None else None,
                            out.handle))
