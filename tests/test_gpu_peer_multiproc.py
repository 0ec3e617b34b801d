"""The peer-memory transport of gscl_jacobi_run across PROCESSES on one GPU.

Two (or three) ranks, one process each, all on cuda:0, no NCCL communicator:
gscl_peer_export / all-gather over gloo / gscl_peer_import, then
gscl_jacobi_run with transport = 1 — boundary planes stored by the pass kernel
into the neighbours' IPC-mapped halo / ghost planes, arrival counters bumped
with system-scope atomics, stream waits on the counters, residual partials
published into every rank's slots.  The processes time-share the GPU, so this
runs slowly, but every cross-rank step of the multi-GPU path runs for real.
Result: the joined slabs equal the oracle's single-domain run bit for bit and
the residual history agrees within 1e-10 — for two consecutive calls (the
second starts with swapped storages and passes the start barrier)."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 12071746


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        import oracle
        from paper_1207_1746_b200 import gscl
        dist.init_process_group("gloo", rank=rank, world_size=world)
        op, nx, ny, nz, iters, check, calls, h, dt = case
        gscl.init(rank, world, device=0, use_nccl=False)
        u = gscl.Grid(nx, ny, nz, h, dt).fill_random(SEED, 0)
        v = gscl.Grid(nx, ny, nz, h, dt)
        cs = [gscl.Grid(nx, ny, nz, 0, dt).fill_random(SEED, 2 + i, 0.125) for i in range(7)] \
            if op == "VARCOEF8" else []

        def gather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        gscl.peer_setup(u, v, gather)
        hists = []
        for _ in range(calls):
            hists.append(gscl.jacobi_run(op, u, v, iters=iters, check_every=check, coeffs=cs))
        # do_reduce across the ranks without NCCL: the peer arena's slots
        red = (gscl.do_reduce("VALUE", [u], "SUM"), gscl.do_reduce("VALUE", [u], "MAX"),
               gscl.do_reduce("RESID7_SQ", [u], "SUM"))
        loc = u.to_host()
        z0 = u.z_begin
        dig = oracle.digest(np.ascontiguousarray(loc), h, z_off=z0)
        digs = gather(dig)
        q.put((rank, sum(digs) % 2 ** 64, hists, red))
        gscl.finalize()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("world,case", [
    (2, ("JACOBI7", 64, 40, 24, 8, 4, 2, 1, 0)),    # 12 planes per rank, checks on pairs
    (3, ("JACOBI7", 40, 33, 27, 7, 3, 2, 1, 0)),    # 9 planes per rank, odd iters / checks: single steps too
    (2, ("JACOBI7", 36, 20, 16, 6, 2, 2, 2, 0)),    # halo 2: both received planes land in the grid
    (2, ("JACOBI7", 70, 33, 20, 6, 2, 1, 1, 1)),    # fp32
    (2, ("JACOBI27", 48, 30, 14, 5, 2, 2, 1, 0)),   # single sweeps, boundary planes stored by the sweep kernel
    (2, ("VARCOEF8", 40, 28, 10, 4, 2, 1, 1, 0)),   # 8 grids read; only u's planes travel (single sweeps)
    (2, ("VARCOEF8", 40, 28, 16, 6, 3, 2, 1, 0)),   # VARCOEF8 two-sweep passes (8 planes per rank)
    (3, ("VARCOEF8", 34, 20, 21, 9, 3, 1, 1, 0)),   # ... 3 ranks, odd-position check sweeps
])
def test_peer_transport_two_processes_one_gpu(world, case):
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
    try:
        res = [q.get(timeout=240) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in res:
        assert r[1] != "error", r[2]
    op, nx, ny, nz, iters, check, calls, h, dt = case
    npdt = np.float64 if dt == 0 else np.float32
    a = oracle.alloc(nx, ny, nz, h, npdt)
    oracle.fill_random(a, h, SEED, 0)
    b = oracle.alloc(nx, ny, nz, h, npdt)
    cs = []
    if op == "VARCOEF8":
        for i in range(7):
            c = oracle.alloc(nx, ny, nz, 0)
            oracle.fill_random(c, 0, SEED, 2 + i, 0.125)
            cs.append(c)
    refs = []
    for _ in range(calls):
        fin, ref = oracle.jacobi_run(op, a, b, h, iters, check, coeffs=cs or None, ch=0)
        if fin is not a:
            a, b = b, a
        refs.append(ref)
    want = oracle.digest(a, h)
    vsum, vabs = oracle.do_reduce("VALUE", [a], [h], "SUM")
    vmax, _ = oracle.do_reduce("VALUE", [a], [h], "MAX")
    rsum, rabs = oracle.do_reduce("RESID7_SQ", [a], [h], "SUM") if h >= 1 else (0.0, 0.0)
    for rank, dig, hists, red in res:
        assert dig == want, f"rank {rank}: joined slabs differ from the single domain"
        assert abs(red[0] - vsum) <= 1e-10 * vabs and red[1] == vmax
        assert abs(red[2] - rsum) <= 1e-10 * rabs
        for h, r in zip(hists, refs):
            assert len(h) == len(r)
            assert all(abs(x - y) <= 1e-10 * y for x, y in zip(h, r)), (h, r)


def _conv_worker(rank, world, port, case, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        import oracle
        from paper_1207_1746_b200 import gscl
        dist.init_process_group("gloo", rank=rank, world_size=world)
        op, nx, ny, nz, eps, maxit, batch = case
        gscl.init(rank, world, device=0, use_nccl=False)
        u = gscl.Grid(nx, ny, nz, 1).fill_random(SEED, 0)
        v = gscl.Grid(nx, ny, nz, 1)

        def gather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        gscl.peer_setup(u, v, gather)
        it, conv = gscl.converge_run(op, u, v, eps, maxit, batch)
        dig = oracle.digest(np.ascontiguousarray(u.to_host()), 1, z_off=u.z_begin)
        q.put((rank, sum(gather(dig)) % 2 ** 64, it, conv))
        gscl.finalize()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("world,case", [
    (2, ("FIG1B", 48, 32, 20, 1e-6, 200, 4)),   # the paper's loop (converges in ~12 iterations)
    (3, ("JACOBI7", 40, 30, 21, 1e-3, 40, 16)),  # max_iters reached, odd batch tail
])
def test_converge_run_peer_transport_processes(world, case):
    # the paper's convergence-terminated loop across ranks with no NCCL: halo
    # planes over IPC + counters, the AND over the peer arena's slots
    import oracle
    oracle.build()
    from paper_1207_1746_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_conv_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=240) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in res:
        assert r[1] != "error", r[2]
    op, nx, ny, nz, eps, maxit, batch = case
    a = oracle.alloc(nx, ny, nz, 1)
    oracle.fill_random(a, 1, SEED, 0)
    fin, it_ref, conv_ref = oracle.converge_run(op, a, oracle.alloc(nx, ny, nz, 1), 1, eps, maxit)
    for rank, dig, it, conv in res:
        assert (it, conv) == (it_ref, conv_ref)
        assert dig == oracle.digest(fin, 1)


def _spawn(target, world, case, timeout=240):
    import oracle
    oracle.build()
    from paper_1207_1746_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = sorted((q.get(timeout=timeout) for _ in range(world)), key=lambda r: r[0])
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in res:
        assert r[1] != "error", r[2]
    return res


def _plane_worker(rank, world, port, case, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        from paper_1207_1746_b200 import gscl
        dist.init_process_group("gloo", rank=rank, world_size=world)
        op, nx, ny, nz, iters, check, h = case
        gscl.init(rank, world, device=0, use_nccl=False)
        u = gscl.Grid(nx, ny, nz, h).fill_random(SEED, 0)
        v = gscl.Grid(nx, ny, nz, h)
        cs = [gscl.Grid(nx, ny, nz, 0).fill_random(SEED, 2 + i, 0.125) for i in range(7)] \
            if op == "VARCOEF8" else []

        def gather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        gscl.peer_setup(u, v, gather)
        gscl.jacobi_run(op, u, v, iters=iters, check_every=check, coeffs=cs)
        dv = u.device_view().cpu().numpy()  # (nzl + 2h, ny + 2h, pitch): the padded local array
        n = u.nzl
        planes = {"halo_lo": dv[0:h].tobytes(), "first": dv[h:2 * h].tobytes(),
                  "last": dv[n:n + h].tobytes(), "halo_hi": dv[n + h:n + 2 * h].tobytes()}
        q.put((rank, planes))
        dist.barrier()
        gscl.finalize()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("world,case", [
    (2, ("JACOBI7", 50, 30, 16, 6, 0, 1)),    # two-sweep passes, no checks
    (3, ("JACOBI7", 40, 24, 21, 5, 5, 1)),    # an unpaired check sweep last (plane copies)
    (2, ("JACOBI7", 36, 20, 16, 4, 2, 2)),    # halo 2: both planes in the grid
    (2, ("JACOBI27", 40, 26, 12, 3, 0, 1)),   # single sweeps: planes stored by the sweep kernel
    (2, ("VARCOEF8", 34, 22, 10, 3, 3, 1)),
    (2, ("VARCOEF8", 34, 22, 14, 4, 0, 1)),   # two-sweep passes (7 planes per rank)
])
def test_peer_halo_planes_equal_neighbour_boundary_planes(world, case):
    # after the exchange each ghost plane IS the
    # neighbour's boundary plane, memcmp-exact — the whole padded xy plane
    # (x / y halo ring and padding included), checked directly rather than
    # through the joined grid's digest
    res = _spawn(_plane_worker, world, case)
    h = case[-1]
    for r in range(world):
        pl = res[r][1]
        if r > 0:
            assert pl["halo_lo"] == res[r - 1][1]["last"], f"rank {r}: lower ghost planes != rank {r-1}'s last {h}"
        if r < world - 1:
            assert pl["halo_hi"] == res[r + 1][1]["first"], f"rank {r}: upper ghost planes != rank {r+1}'s first {h}"


def _timeout_worker(rank, world, port, case, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import time
        import torch.distributed as dist
        from paper_1207_1746_b200 import gscl
        dist.init_process_group("gloo", rank=rank, world_size=world)
        op, check = case
        gscl.init(rank, world, device=0, use_nccl=False)
        u = gscl.Grid(48, 32, 16, 1).fill_random(SEED, 0)
        v = gscl.Grid(48, 32, 16, 1)

        def gather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        gscl.peer_setup(u, v, gather)
        if rank == world - 1:  # the "missing" rank: never calls jacobi_run
            dist.barrier()
            gscl.finalize()
            q.put((rank, "idle"))
        else:
            gscl.set_option("timeout_ms", 2000)
            t0 = time.time()
            try:
                if op == "CONVERGE":
                    gscl.converge_run("FIG1B", u, v, 1e-6, 50, 4)
                elif op == "REDUCE":
                    gscl.do_reduce("VALUE", [u], "SUM")
                elif op == "DIGEST":
                    u.digest()
                else:
                    gscl.jacobi_run(op, u, v, iters=6, check_every=check)
                status = "no error"
            except gscl.GsclError as e:
                status = e.name
            dt = time.time() - t0
            try:
                gscl.do_reduce("VALUE", [u], "SUM")
                after = "no error"
            except gscl.GsclError as e:
                after = e.name
            fin = "ok"
            try:
                gscl.finalize()
            except gscl.GsclError as e:
                fin = e.name
            q.put((rank, status, dt, after, fin))
            dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("case", [("JACOBI7", 2), ("JACOBI7", 0), ("JACOBI27", 3), ("CONVERGE", 0),
                                  ("REDUCE", 0), ("DIGEST", 0)])
def test_peer_missing_rank_times_out_cleanly(case):
    # the multi-rank watchdog: a rank that never joins makes its neighbour's
    # call fail with GSCL_E_TIMEOUT within seconds (option timeout_ms = 2 s)
    # instead of hanging on the counter waits; the context is then poisoned
    # (later calls GSCL_E_STATE) and finalize still returns
    res = _spawn(_timeout_worker, 2, case, timeout=120)
    r0 = res[0]
    assert r0[1] == "GSCL_E_TIMEOUT", r0
    assert r0[2] < 20.0, f"took {r0[2]:.1f} s"
    assert r0[3] == "GSCL_E_STATE" and r0[4] == "ok", r0


def _xchg_worker(rank, world, port, case, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        from paper_1207_1746_b200 import gscl
        dist.init_process_group("gloo", rank=rank, world_size=world)
        nx, ny, nz, h = case
        gscl.init(rank, world, device=0, use_nccl=False)
        u = gscl.Grid(nx, ny, nz, h).fill_random(SEED, 0)
        v = gscl.Grid(nx, ny, nz, h)

        def gather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        gscl.peer_setup(u, v, gather)
        u.fill_random(SEED + 1 + rank, 0)  # different data than at setup: the exchange must move it
        gscl.halo_exchange_depth([u], 2)
        gscl.sync()
        dv = u.device_view().cpu().numpy()
        n = u.nzl
        q.put((rank, {"halo_lo": dv[0:h].tobytes(), "first": dv[h:2 * h].tobytes(),
                      "last": dv[n:n + h].tobytes(), "halo_hi": dv[n + h:n + 2 * h].tobytes()}))
        dist.barrier()
        gscl.finalize()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("world,case", [(2, (40, 24, 14, 1)), (3, (36, 20, 21, 2))])
def test_peer_halo_exchange_depth_moves_boundary_planes(world, case):
    # gscl_halo_exchange_depth over the peer transport (the exchange bench.py
    # times alone): afterwards each halo plane IS the neighbour's boundary
    # plane, memcmp-exact
    res = _spawn(_xchg_worker, world, case)
    h = case[-1]
    for r in range(world):
        pl = res[r][1]
        if r > 0:
            assert pl["halo_lo"] == res[r - 1][1]["last"]
        if r < world - 1:
            assert pl["halo_hi"] == res[r + 1][1]["first"]
