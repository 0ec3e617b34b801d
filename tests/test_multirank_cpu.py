"""Multi-rank host logic on CPU (gloo, world size 2 and 3): the product's own
z-slab split and halo-exchange plan (gscl_slab_range / gscl_halo_plan, the same
ops gscl_halo_exchange issues through NCCL) executed over torch.distributed
gloo on slabs laid out exactly as on the GPU, with the oracle as the sweep.
P-slab results must equal the single-domain oracle bit for bit,
and the rank-order fold of per-rank partial sums (R14) must match the
single-domain reduction within 1e-10."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 12071746


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _padded(lay, dtype=np.float64):
    buf = np.zeros(lay["bytes"], dtype=np.uint8)
    arr = buf.view(dtype).reshape(lay["planes"], lay["rows"], lay["pitch"])
    return buf, arr


def _worker(rank, world, port, case, q):
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        import oracle
        from paper_1207_1746_b200 import gscl
        dist.init_process_group("gloo", rank=rank, world_size=world)
        op, nx, ny, nz, h, iters = case
        # 1) the NCCL unique-id bootstrap gscl.init performs, over gloo
        t = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            t[:] = torch.frombuffer(bytearray(gscl.get_nccl_unique_id()), dtype=torch.uint8)
        dist.broadcast(t, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, bytes(t.numpy().tobytes()))
        assert all(i == ids[0] for i in ids)
        # 2) slabs in the GPU layout, filled by the oracle's generator at global z
        lay = gscl.layout_of(nx, ny, nz, h, gscl.F64, rank, world)
        z0, z1 = lay["z_begin"], lay["z_end"]
        ox = lay["ox"]
        plan = gscl.halo_plan(nx, ny, nz, h, gscl.F64, rank, world)
        ubuf, u = _padded(lay)
        vbuf, v = _padded(lay)
        dense = oracle.alloc(nx, ny, z1 - z0, h)
        oracle.fill_random(dense, h, SEED, 0, z_off=z0)
        u[:, :, ox - h:ox + nx + h] = dense
        v[:, :, ox - h:ox + nx + h] = dense  # the halo shell travels with both buffers
        def exchange(buf):
            reqs = []
            for peer, is_send, off, nb in plan:
                ten = torch.from_numpy(buf[off:off + nb])
                reqs.append(dist.isend(ten, peer) if is_send else dist.irecv(ten, peer))
            for r in reqs:
                r.wait()

        for _ in range(iters):
            exchange(ubuf)
            din = np.ascontiguousarray(u[:, :, ox - h:ox + nx + h])
            dout = np.ascontiguousarray(v[:, :, ox - h:ox + nx + h])
            oracle.do_all(op, [din], [h], dout, h)
            v[:, :, ox - h:ox + nx + h] = dout
            ubuf, vbuf, u, v = vbuf, ubuf, v, u
        exchange(ubuf)  # the final residual reads ghost planes too (as gscl_jacobi_run does)
        final = np.ascontiguousarray(u[:, :, ox - h:ox + nx + h])
        dig = oracle.digest(final, h, z_off=z0)
        resid, asum = oracle.do_reduce("RESID7_SQ", [final], [h], "SUM")
        digs = [None] * world
        dist.all_gather_object(digs, dig)
        parts = [None] * world
        dist.all_gather_object(parts, (resid, asum))
        total = 0.0
        for r_, _ in parts:  # fold in rank order (R14)
            total += r_
        q.put((rank, sum(digs) % 2 ** 64, total, sum(a for _, a in parts), plan, (z0, z1)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("world,case", [
    (2, ("JACOBI7", 13, 11, 17, 1, 4)),
    (2, ("JACOBI27", 12, 9, 10, 1, 3)),
    (3, ("JACOBI7", 9, 8, 11, 1, 3)),
    (2, ("JACOBI7", 10, 7, 9, 2, 2)),   # halo 2: two planes per exchange
])
def test_multirank_slabs_equal_single_domain(world, case):
    import oracle
    oracle.build()
    from paper_1207_1746_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r[2]
    op, nx, ny, nz, h, iters = case
    ref = oracle.alloc(nx, ny, nz, h)
    oracle.fill_random(ref, h, SEED, 0)
    for _ in range(iters):
        out = ref.copy()
        oracle.do_all(op, [ref], [h], out, h)
        ref = out
    d_ref = oracle.digest(ref, h)
    r_ref, a_ref = oracle.do_reduce("RESID7_SQ", [ref], [h], "SUM")
    for rank, dig, total, asum, plan, (z0, z1) in res:
        assert dig == d_ref, "P-slab result differs from the single domain"
        assert abs(total - r_ref) <= 1e-10 * a_ref
        # plan shape: interior ranks exchange with both neighbours
        peers = sorted({p for p, *_ in plan})
        expect = [x for x in (rank - 1, rank + 1) if 0 <= x < world]
        assert peers == expect


def test_halo_plan_offsets():
    from paper_1207_1746_b200 import build
    build.build()
    from paper_1207_1746_b200 import gscl
    nx, ny, nz, h, P = 512, 512, 1024, 1, 2
    lay0 = gscl.layout_of(nx, ny, nz, h, gscl.F64, 0, P)
    plane = lay0["pitch"] * lay0["rows"] * 8
    assert plane == 544 * 514 * 8  # 2.24 MB per exchanged plane
    p0 = gscl.halo_plan(nx, ny, nz, h, gscl.F64, 0, P)
    p1 = gscl.halo_plan(nx, ny, nz, h, gscl.F64, 1, P)
    # rank 0 sends its last interior plane (local 511 -> byte (511+1)*plane) and
    # receives into ghost plane 512 -> byte 513*plane; rank 1 mirrors it.
    assert p0 == [(1, 1, 512 * plane, plane), (1, 0, 513 * plane, plane)]
    assert p1 == [(0, 1, plane, plane), (0, 0, 0, plane)]
    assert gscl.halo_plan(nx, ny, 512, h, gscl.F64, 0, 1) == []
    mid = gscl.halo_plan(64, 64, 96, 2, gscl.F32, 1, 3)
    assert [(p, s) for p, s, _, _ in mid] == [(0, 1), (0, 0), (2, 1), (2, 0)]


def _pass_worker(rank, world, port, case, q):
    """Two-sweep passes (the multi-rank temporal-blocking schedule of
    gscl_jacobi_run) with the product's depth-2 exchange plan (gscl_pass_plan)
    run over gloo; the pass itself is the oracle: u1 = JACOBI7(u) on planes
    -1..nzl of the slab (Dirichlet rule only at physical z ends), then
    out = JACOBI7(u1) on the interior."""
    try:
        sys.path.insert(0, ROOT)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        import oracle
        from paper_1207_1746_b200 import gscl
        dist.init_process_group("gloo", rank=rank, world_size=world)
        nx, ny, nz, h, passes = case
        lay = gscl.layout_of(nx, ny, nz, h, gscl.F64, rank, world)
        z0, z1 = lay["z_begin"], lay["z_end"]
        nzl, ox = z1 - z0, lay["ox"]
        plan = gscl.pass_plan(nx, ny, nz, h, gscl.F64, rank, world)
        ubuf, u = _padded(lay)
        vbuf, v = _padded(lay)
        ghost = np.zeros((2, lay["rows"], lay["pitch"]))
        dense = oracle.alloc(nx, ny, nzl, h)
        oracle.fill_random(dense, h, SEED, 0, z_off=z0)
        u[:, :, ox - h:ox + nx + h] = dense
        v[:, :, ox - h:ox + nx + h] = dense

        def plane(arr, z, gp):
            return ghost[gp - 1] if gp else arr[z + h]

        def exchange(arr):
            reqs = []
            for peer, is_send, z, gp in plan:
                buf = plane(arr, z, gp)
                ten = torch.from_numpy(buf.reshape(-1))
                reqs.append(dist.isend(ten, peer) if is_send else dist.irecv(ten, peer))
            for r_ in reqs:
                r_.wait()

        lo_phys, hi_phys = rank == 0, rank == world - 1
        for _ in range(passes):
            exchange(u)
            # planes -2 .. nzl+1 of u as a dense (nzl+4, ny+2h, nx+2h) array
            ext = np.zeros((nzl + 4, ny + 2 * h, nx + 2 * h))
            for k, z in enumerate(range(-2, nzl + 2)):
                if -h <= z < nzl + h:
                    src = u[z + h]
                elif z < 0:
                    src = ghost[0] if not lo_phys else np.zeros_like(u[0])
                else:
                    src = ghost[1] if not hi_phys else np.zeros_like(u[0])
                ext[k] = src[:, ox - h:ox + nx + h]
            # u1 on planes -1..nzl: ext as an h=1 grid (z) whose interior is those planes;
            # x/y halo width h >= 1 — use a halo-1 view of the x/y extent
            e1 = np.ascontiguousarray(ext[:, h - 1:ny + h + 1, h - 1:nx + h + 1])
            u1 = e1.copy()
            oracle.do_all("JACOBI7", [e1], [1], u1, 1)
            if lo_phys:
                u1[1] = e1[1]   # plane -1 is the Dirichlet boundary
            if hi_phys:
                u1[nzl + 2] = e1[nzl + 2]
            w = np.ascontiguousarray(u1[1:nzl + 3])   # planes -1..nzl = h=1 grid of nzl
            out = w.copy()
            oracle.do_all("JACOBI7", [w], [1], out, 1)
            v[h:h + nzl, h:h + ny, ox:ox + nx] = out[1:1 + nzl, 1:1 + ny, 1:1 + nx]
            ubuf, vbuf, u, v = vbuf, ubuf, v, u
        final = np.ascontiguousarray(u[:, :, ox - h:ox + nx + h])
        dig = oracle.digest(final, h, z_off=z0)
        digs = [None] * world
        dist.all_gather_object(digs, dig)
        q.put((rank, sum(digs) % 2 ** 64, plan))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("world,case", [
    (2, (11, 9, 14, 1, 3)),
    (3, (9, 10, 13, 1, 2)),
    (2, (8, 7, 9, 2, 2)),     # halo 2: both received planes land in the grid
    (3, (7, 6, 6, 1, 2)),     # 2 planes per rank: every plane is a boundary plane
])
def test_multirank_two_sweep_passes_equal_single_domain(world, case):
    import oracle
    oracle.build()
    from paper_1207_1746_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pass_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r[2]
    nx, ny, nz, h, passes = case
    ref = oracle.alloc(nx, ny, nz, h)
    oracle.fill_random(ref, h, SEED, 0)
    for _ in range(2 * passes):
        out = ref.copy()
        oracle.do_all("JACOBI7", [ref], [h], out, h)
        ref = out
    for rank, dig, plan in res:
        assert dig == oracle.digest(ref, h), f"rank {rank}: P-slab passes differ from 2x{passes} sweeps"


def test_pass_plan_shape():
    from paper_1207_1746_b200 import build
    build.build()
    from paper_1207_1746_b200 import gscl
    n = 7  # nz 20 over 3 ranks: 7, 7, 6 planes
    assert gscl.pass_plan(8, 8, 20, 1, gscl.F64, 0, 3) == [(1, 1, n - 1, 0), (1, 1, n - 2, 0),
                                                          (1, 0, n, 0), (1, 0, n + 1, 2)]
    assert gscl.pass_plan(8, 8, 20, 1, gscl.F64, 2, 3) == [(1, 1, 0, 0), (1, 1, 1, 0),
                                                          (1, 0, -1, 0), (1, 0, -2, 1)]
    # halo 2: the second plane is in the grid's own halo
    assert [g for *_, g in gscl.pass_plan(8, 8, 20, 2, gscl.F64, 1, 3)] == [0] * 8
    assert gscl.pass_plan(8, 8, 20, 1, gscl.F64, 0, 1) == []
    with pytest.raises(gscl.GsclError):
        gscl.pass_plan(8, 8, 3, 1, gscl.F64, 0, 3)  # 1 plane per rank
