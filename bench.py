#!/usr/bin/env python
"""bench.py — the headline measurement.

Workload (BASELINE.json `configs`): one step = one gscl_jacobi_run of the
7-point Laplacian Jacobi operator (JACOBI7), fp64, 512^3 interior + halo 1 per
GPU, 100 sweeps with the L2 residual fused into every 10th sweep plus a final
residual pass — config 2 at N=1; config 5 (weak scaling, global nz = 512*N,
z-slabs, halo exchange + cross-rank combine) at N>1.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--n 512]

Prints ONE JSON line on rank 0.  `value` is whole-job Gpoint-updates/s from
CUDA events on the library stream (max over ranks); `e2e` is the same metric
through the public API with the initial grid copied from pinned host memory
and the residual history read back every step (`e2e.with_final_iterate`: the
final iterate copied back too); `roofline` is the dominant kernel against
MEASURED_PEAKS.json; `cpu_baseline` is the CPU oracle on a bounded sample
(rank 0, N=1 only).  At N>1 the line adds `halo` (exchange-only and exposed
halo time for the NCCL and the peer-memory transports) and `parity` (the
joined slabs' digest and residual history against a single-domain run of the
same global grid on rank 0's GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpoint-updates/s and achieved HBM GB/s vs peak, at 1/2/4/8 B200"
UNIT = "Gpoint-updates/s"
SEED = 12071746
BYTES_PER_PT = 16.0  # JACOBI7 fp64: read u once, write v once
L2_BYTES = 126 * 2 ** 20


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic(key="jacobi7_pass"):
    """dram bytes per launch of a kernel from the committed ncu capture
    (jacobi7_pass: the two-sweep pass; jacobi7_sweep: the do_all sweep)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return j.get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class Clocks:
    """Sample SM clocks and clock-event (throttle) reasons DURING the timed
    region.  Primary: an in-process NVML thread (the library nvidia-smi reads)
    polling every 5 ms from the moment the region starts to the moment it
    ends — an `nvidia-smi -lms` child needs a few hundred ms to start and gave
    0-4 samples of a ~0.2 s region.  Fallback (no NVML): the recipe's
    `nvidia-smi ... -lms 20` loop across the region plus a one-shot query."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,clocks.mem,power.draw")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    # NVML clock-event reason bits for NAMES
    BITS = [0x8, 0x40, 0x20, 0x4]

    def __init__(self, device: int, period_ms: int = 20, nvml_period_ms: float = 5.0):
        self.device = device
        self.period_ms = period_ms
        self.nvml_period = nvml_period_ms / 1e3
        self.samples = []
        self._p = None
        self._t = None
        self._stop = None
        self.source = f"nvidia-smi -lms {period_ms}"

    def _cmd(self, loop: bool):
        c = ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"]
        return c + ["-lms", str(self.period_ms)] if loop else c

    def _parse(self, text: str):
        for line in text.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                extra = (float(f[6]) if len(f) > 6 else float("nan"), float(f[7]) if len(f) > 7 else float("nan"))
            except ValueError:
                extra = (float("nan"), float("nan"))
            try:
                self.samples.append((float(f[0]), float(f[1]),
                                     {self.NAMES[i] for i in range(4) if f[i + 2].lower() == "active"}) + extra)
            except ValueError:
                pass

    def _nvml_start(self) -> bool:
        try:
            import threading

            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def one():
                r = reasons(h)
                try:
                    pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                except Exception:
                    pw = float("nan")
                return (float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), float(smax),
                        {self.NAMES[i] for i in range(4) if r & self.BITS[i]},
                        float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM)), pw)

            one()  # fail here, not in the thread
            self._stop = threading.Event()

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append(one())
                    except Exception:
                        pass
                    self._stop.wait(self.nvml_period)
                try:
                    self.samples.append(one())  # the region's last moment
                except Exception:
                    pass

            self._t = threading.Thread(target=loop, daemon=True)
            self._t.start()
            self.source = f"NVML in-process, every {self.nvml_period * 1e3:.0f} ms"
            return True
        except Exception:
            return False

    def __enter__(self):
        if self._nvml_start():
            return self
        try:
            self._p = subprocess.Popen(self._cmd(True), stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                       text=True)
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._t is not None:
            self._stop.set()
            self._t.join(timeout=5)
            return
        if self._p is not None:
            try:
                self._p.terminate()
                out, _ = self._p.communicate(timeout=5)
                self._parse(out)
            except Exception:
                try:
                    self._p.kill()
                except Exception:
                    pass
        try:
            self._parse(subprocess.run(self._cmd(False), capture_output=True, text=True,
                                       timeout=5).stdout)
        except Exception:
            pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        mem = [s[3] for s in self.samples if len(s) > 3 and s[3] == s[3]]
        pw = [s[4] for s in self.samples if len(s) > 4 and s[4] == s[4]]
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "sm_mhz_min": min(s[0] for s in self.samples),
                "reasons": sorted(set().union(*(s[2] for s in self.samples))),
                "mem_mhz": statistics.median(mem) if mem else None,
                "power_w_median": statistics.median(pw) if pw else None,
                "samples": len(self.samples), "source": self.source}


# ---------------------------------------------------------------- CPU oracle legs
def _oracle_run(n: int, sweeps: int, check: int):
    """Time the CPU oracle (as it stands) on `sweeps` JACOBI7 sweeps of n^3
    with the residual every `check` sweeps (+ the final residual)."""
    import oracle
    oracle.build()
    u = oracle.alloc(n, n, n, 1)
    oracle.fill_random(u, 1, SEED, 0)
    v = oracle.alloc(n, n, n, 1)
    t0 = time.perf_counter()
    oracle.jacobi_run("JACOBI7", u, v, 1, sweeps, check)
    return time.perf_counter() - t0


def cpu_baseline(n: int) -> dict:
    """The oracle on the box's host cores: all cores (OpenMP over z, the
    reported value) and one thread, on bounded samples of the config-2 step;
    per-element ns as the paper reports it (time / elements /
    iterations); config 1 (32^3, 10 sweeps, residual every sweep) in seconds."""
    import oracle
    oracle.build()
    cores = oracle.num_threads()
    _oracle_run(n, 1, 1)  # warm (page-in, thread pool)
    dt2 = _oracle_run(n, 2, 2)
    sweeps = max(2, min(400, int(12.0 / max(dt2 / 2, 1e-3))))  # ~12 s of all-core oracle work
    dt = _oracle_run(n, sweeps, sweeps)
    val = n ** 3 * sweeps / dt / 1e9
    c1_all = min(_oracle_run(32, 10, 1) for _ in range(3))
    oracle.set_threads(1)
    try:
        d1 = _oracle_run(n, 1, 0)
        s1 = max(1, min(20, int(6.0 / max(d1, 1e-3))))  # ~6 s of one-thread work
        dt1 = _oracle_run(n, s1, 0)  # (sweeps only: at this sample size the residual pass would dominate)
        c1_one = min(_oracle_run(32, 10, 1) for _ in range(3))
    finally:
        oracle.set_threads(cores)
    v1 = n ** 3 * s1 / dt1 / 1e9
    return {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"JACOBI7 fp64 {n}^3: all cores {sweeps} sweeps + residual ({dt:.2f} s); one thread "
                      f"{s1} sweeps, no residual ({dt1:.2f} s); the timed GPU step has 100 sweeps",
            "cpu_model": _cpu_model(),
            "ns_per_point_update": 1e9 * dt / (n ** 3 * sweeps),
            "one_thread": {"value": v1, "unit": UNIT, "ns_per_point_update": 1e9 * dt1 / (n ** 3 * s1)},
            "config1_seconds": {"all_cores": c1_all, "one_thread": c1_one,
                                "what": "JACOBI7 fp64 32^3 + halo 1, 10 sweeps, residual every sweep + final"}}


def run_reference(args, rank: int, world: int):
    """--impl reference: the CPU oracle is this tier's reference arm."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    n = args.n
    u = oracle.alloc(n, n, n, 1)
    oracle.fill_random(u, 1, SEED, 0)
    v = oracle.alloc(n, n, n, 1)
    iters = args.ref_iters
    for _ in range(args.warmup):
        oracle.jacobi_run("JACOBI7", u, v, 1, iters, iters)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.jacobi_run("JACOBI7", u, v, 1, iters, iters)
    dt = time.perf_counter() - t0
    pts = n ** 3 * iters * args.steps * world
    val = pts / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (splitmix64 U[0,1) interior, zero Dirichlet halo)",
        "config": {"workload": f"config{2 if world == 1 else 5}: JACOBI7 fp64 {n}^3 per GPU; "
                               f"reference step = {iters} sweeps + fused/final residual "
                               f"(bounded sample of the 100-sweep step)"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle.num_threads(),
                         "kind": "oracle", "cpu_model": _cpu_model(),
                         "sample": f"{iters} JACOBI7 sweeps of {n}^3 per step, {args.steps} steps"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _bind_to_gpu_numa_node(device: int) -> str:
    """Pin this process to the CPUs of the GPU's NUMA node (sysfs local_cpulist),
    so pinned host buffers are first-touched on the node next to the GPU's PCIe
    root (the e2e uploads) and launches run on near cores.  Best effort."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(device)
        bus = (f"{int(getattr(pr, 'pci_domain_id', 0)):04x}:{int(pr.pci_bus_id):02x}:"
               f"{int(getattr(pr, 'pci_device_id', 0)):02x}.0")
        path = f"/sys/bus/pci/devices/{bus}/local_cpulist"
        txt = open(path).read().strip()
        cpus = set()
        for part in txt.split(","):
            if "-" in part:
                lo, hi = part.split("-")
                cpus.update(range(int(lo), int(hi) + 1))
            elif part:
                cpus.add(int(part))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return txt
    except Exception:
        pass
    return "unbound"


def run_single_domain(args):
    """--single-domain (a child of rank 0 at N>1): the whole global grid
    n x n x nz on ONE GPU, one bench step from the seeded input; prints
    {"digest", "hist"} — the reference the joined slabs must equal."""
    import torch
    from paper_1207_1746_b200 import gscl
    torch.cuda.set_device(0)
    gscl.init(0, 1, device=0)
    n, nz = args.n, args.single_domain
    u = gscl.Grid(n, n, nz, 1).fill_random(SEED, 0)
    v = gscl.Grid(n, n, nz, 1)
    hist = gscl.jacobi_run("JACOBI7", u, v, iters=args.iters, check_every=args.check_every)
    print(json.dumps({"digest": u.digest(), "hist": hist}), flush=True)
    gscl.finalize()


def run_gpu(args, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch

    one_gpu = args.one_gpu_ranks and world > 1  # debug: every rank on GPU 0, no NCCL
    if one_gpu:
        local_rank = 0
    if world > 1:
        # the library's NCCL communicator logs its init lines (rank / nranks checkable)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # (stdout carries the one JSON line)
    torch.cuda.set_device(local_rank)
    all_cpus = os.sched_getaffinity(0)
    numa_cpus = _bind_to_gpu_numa_node(local_rank)
    dist = None
    if world > 1:
        # host-side coordination only (barriers, max over ranks, id broadcast,
        # blob gathers) over gloo; the data path's collectives are the library's
        import torch.distributed as dist
        dist.init_process_group("gloo")
    from paper_1207_1746_b200 import gscl

    def max_over_ranks(xs):
        """element-wise max over ranks of a list of floats (gloo, host)."""
        if dist is None:
            return list(xs)
        t = torch.tensor(list(xs), dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def gather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    nccl_id = None
    if world > 1 and not one_gpu:
        obj = [gscl.get_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    gscl.init(rank, world, device=local_rank, nccl_id=nccl_id, use_nccl=not one_gpu)
    if world > 1:
        gscl.set_option("timeout_ms", args.timeout_ms)

    n = args.n
    nz = n * world
    iters, check = args.iters, args.check_every
    u = gscl.Grid(n, n, nz, 1).fill_random(SEED, 0)
    v = gscl.Grid(n, n, nz, 1)
    stream = torch.cuda.current_stream()
    # headline transport at N>1: NCCL send/recv (the north star's); the
    # peer-memory transport is measured beside it (`halo.p2p`)
    transport = "none" if world == 1 else ("p2p" if one_gpu else "nccl")
    peer_ok, peer_err = False, None

    def setup_peer():
        nonlocal peer_ok, peer_err
        try:
            gscl.peer_setup(u, v, gather)
            peer_ok = True
        except Exception as ex:  # every rank sees the same failure mode
            peer_err = str(ex)[:200]
            gscl.set_option("transport", 0)
        return peer_ok

    if one_gpu:
        if not setup_peer():
            raise RuntimeError(f"--one-gpu-ranks needs the peer transport: {peer_err}")

    def barrier():
        if dist is not None:
            dist.barrier()

    def step():
        return gscl.jacobi_run("JACOBI7", u, v, iters=iters, check_every=check)

    def timed_steps(nsteps):
        """nsteps timed steps: CUDA events on the library stream around every
        step, barrier + synchronize on both sides, max over ranks; the
        library's kernel timing on (events around each sweep launch, one
        pair around each run of consecutive two-sweep passes)."""
        gscl.timing_read()
        gscl.timing_enable(True)
        barrier()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(nsteps + 1)]
        evs[0].record(stream)
        h = None
        for k in range(nsteps):
            h = step()
            evs[k + 1].record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_k, n_k, launches = gscl.timing_read()
        gscl.timing_enable(False)
        per = [evs[k].elapsed_time(evs[k + 1]) for k in range(nsteps)]
        allm = max_over_ranks([evs[0].elapsed_time(evs[-1])] + per)
        return allm[0], allm[1:], ms_k, n_k, launches, h

    for _ in range(args.warmup):
        step()
    with Clocks(local_rank, args.clock_ms) as clk:
        elapsed, per_step, ms_k, n_k, launches, hist = timed_steps(args.steps)
    ms_per_step = elapsed / args.steps
    pts_step = float(n) * n * nz * iters
    value = pts_step / (ms_per_step * 1e-3) / 1e9

    peak, peak_kind = _peaks()

    def copy_gbs() -> float:
        """Same-box reference: torch copy_ of 1 GiB (best of 5), read + write bytes."""
        try:
            src = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
            dst = torch.empty_like(src)
            dst.copy_(src)
            best = 1e30
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dst.copy_(src)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            del src, dst
            torch.cuda.empty_cache()
            return 2.0 * (1 << 30) / (best * 1e-3) / 1e9
        except Exception:
            return float("nan")
    local_pts = float(n) * n * (u.nzl)
    step_share = sum(ms_k) / max(elapsed, 1e-9)

    def sweep_roofline(ms_k, n_k, nsteps):
        """the do_all JACOBI7 sweep (kind 0).  On several ranks a sweep is split
        into boundary + interior launches, so average over the number of
        whole-slab sweeps they make up (iters - checks per step)."""
        sweeps_k0 = nsteps * (iters - (iters // check if check > 0 else 0))
        avg = ms_k[0] / max(sweeps_k0, 1)
        ach = BYTES_PER_PT * local_pts / (avg * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": _traffic("jacobi7_sweep"), "kernel": "sweep_tma<JACOBI7> (do_all, one sweep)",
                "peak_kind": peak_kind, "bytes_per_launch": BYTES_PER_PT * local_pts,
                "avg_launch_ms": avg, "sweep_launches": n_k[0], "frac_of_8TBs": ach / 8000.0,
                "fused_avg_launch_ms": ms_k[1] / max(n_k[1], 1)}

    # the dominant kernel.  Default schedule: the two-sweep pass (kind 3,
    # sweep2r_tma: 100 sweeps = 50 passes, the residual of every 10th sweep
    # fused into its pass); algorithmic bytes per pass = 16 B/pt (read u,
    # write the iterate two sweeps later).  Otherwise the do_all sweep.
    if n_k[3] > 0:
        pass_ms = ms_k[3] / n_k[3]
        achieved = BYTES_PER_PT * local_pts / (pass_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": _traffic("jacobi7_pass"),
                "kernel": "sweep2r_tma<JACOBI7> (two sweeps per HBM pass, temporal blocking)",
                "peak_kind": peak_kind, "bytes_per_launch": BYTES_PER_PT * local_pts,
                "avg_launch_ms": pass_ms, "pass_launches": n_k[3], "frac_of_8TBs": achieved / 8000.0,
                "sweep_equiv_GBps": 2 * achieved, "pass_share_of_step": ms_k[3] / max(elapsed, 1e-9)}
    else:
        roof = sweep_roofline(ms_k, n_k, args.steps)
    roof["timed_share_of_step"] = step_share
    if world == 1:  # context beside `peak`: the same box's copy bandwidth, measured now
        cg = copy_gbs()
        roof["copy_gbs_same_box"] = cg
        roof["frac_of_same_box_copy"] = roof["achieved"] / cg if cg == cg else None

    # ---- the same step with one sweep per HBM pass (tblock = 1): the do_all
    # sweep kernel against the roofline (reported beside the default schedule)
    single = None
    if world == 1 and n_k[3] > 0 and not args.no_next2:
        gscl.set_option("tblock", 1)
        for _ in range(2):
            step()
        nsteps = max(1, min(args.steps, 5))
        t1, _, ms1k, n1k, _, _ = timed_steps(nsteps)
        gscl.set_option("tblock", 0)
        single = {"what": "same step, one sweep per HBM pass (gscl_set_option tblock=1)",
                  "value": pts_step / (t1 / nsteps * 1e-3) / 1e9, "unit": UNIT,
                  "ms_per_step": t1 / nsteps, "roofline": sweep_roofline(ms1k, n1k, nsteps)}

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a0.record(stream)
        for _ in range(reps):
            fn()
        a1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks([a0.elapsed_time(a1) / reps])[0]

    # ---- N > 1: halo time reported separately: the exchange
    # alone, and exposed = overlapped step - compute-only step (halo_off)
    halo = None
    if world > 1:
        halo = {"planes_per_side_per_pass": 2, "plane_bytes": u.pitch * (n + 2) * 8,
                "passes_per_step": iters // 2}
        gscl.set_option("halo_off", 1)
        try:
            t_comp = timed(step, max(2, min(args.steps, 5)))
        finally:
            gscl.set_option("halo_off", 0)
        halo["compute_only_ms_per_step"] = t_comp
        reps = 50

        def xchg_ms(depth):
            return timed(lambda: gscl.halo_exchange_depth([u], depth), reps)
        # the headline transport's numbers (NCCL; the peer transport with --one-gpu-ranks)
        hk = "nccl" if not one_gpu else "p2p"
        halo[hk] = {"step_ms": ms_per_step,
                    "exchange_only_ms": {"depth2": xchg_ms(2)} if one_gpu else
                                        {"depth2": xchg_ms(2), "depth1": xchg_ms(1)},
                    "exposed_ms_per_step": ms_per_step - t_comp,
                    "exposed_ms_per_pass": (ms_per_step - t_comp) / (iters // 2)}

    # ---- N > 1: self-verification.  The joined slabs after one step from the
    # seeded input must equal a single-domain run of the same global grid
    # (rank 0's GPU, a child process): digest bitwise, history within 1e-10.
    parity = None
    parity_ref = None
    if world > 1 and not args.no_parity:
        parity = {"reference": f"single-domain {n}x{n}x{nz} on one GPU (child process of rank 0)"}
        runs = [("nccl", 0)] if not one_gpu else [("p2p", 1)]
        got = {}
        for name, tr in runs:
            try:
                gscl.set_option("transport", tr)
                u.fill_random(SEED, 0)
                hh = step()
                got[name] = (u.digest(), hh)
            except Exception as ex:
                got[name] = (None, str(ex)[:200])
        gscl.set_option("transport", 1 if one_gpu else 0)
        ref = None
        if rank == 0:
            env = dict(os.environ)
            env["CUDA_VISIBLE_DEVICES"] = env.get("CUDA_VISIBLE_DEVICES", "").split(",")[local_rank] \
                if env.get("CUDA_VISIBLE_DEVICES") else str(local_rank)
            for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "GROUP_RANK", "ROLE_RANK",
                      "ROLE_WORLD_SIZE", "TORCHELASTIC_RUN_ID", "NCCL_DEBUG"):
                env.pop(k, None)
            try:
                out = subprocess.run([sys.executable, os.path.abspath(__file__), "--single-domain", str(nz),
                                      "--n", str(n), "--iters", str(iters), "--check-every", str(check)],
                                     env=env, capture_output=True, text=True, timeout=600)
                ref = json.loads(out.stdout.strip().splitlines()[-1])
            except Exception as ex:
                parity["error"] = f"single-domain run failed: {str(ex)[:200]}"
        barrier()
        if rank == 0 and ref is not None:
            ok_all = True
            for name, (dg, hh) in got.items():
                if dg is None:
                    parity[name] = {"ok": False, "error": hh}
                    ok_all = False
                    continue
                rel = max((abs(a - b) / max(abs(b), 1e-300) for a, b in zip(hh, ref["hist"])), default=0.0)
                ok = dg == ref["digest"] and len(hh) == len(ref["hist"]) and rel <= 1e-10
                parity[name] = {"ok": ok, "digest": f"{dg:016x}", "hist_max_rel": rel}
                ok_all &= ok
            parity["single_domain_digest"] = f"{ref['digest']:016x}"
            parity["parity_ok"] = ok_all and bool(got)
            parity_ref = ref
        elif rank == 0:
            parity["parity_ok"] = False

    # ---- the other BASELINE configs on this GPU (N = 1 only; bounded, device-timed)
    others = None
    if world == 1 and not args.no_configs:
        others = {}
        # config 1: 7-point Jacobi fp64 32^3 + halo 1, 10 iterations, L2 residual every iteration
        c1u = gscl.Grid(32, 32, 32, 1).fill_random(SEED, 0)
        c1v = gscl.Grid(32, 32, 32, 1)
        ms1 = timed(lambda: gscl.jacobi_run("JACOBI7", c1u, c1v, iters=10, check_every=1), 50)
        others["config1_jacobi7_32cubed"] = {"ms_per_run": ms1, "Gpts": 32 ** 3 * 10 / ms1 / 1e6,
                                             "note": "10 sweeps + 11 residuals, one CUDA graph"}
        c1u.destroy(); c1v.destroy()
        # config 3: 27-point Jacobi fp64 512^3, 100 sweeps, residual every 10
        ms3 = timed(lambda: gscl.jacobi_run("JACOBI27", u, v, iters=iters, check_every=check), 2)
        others["config3_jacobi27_512cubed"] = {"ms_per_step": ms3, "Gpts": pts_step / ms3 / 1e6,
                                               "hbm_gbs_algorithmic": BYTES_PER_PT * pts_step / ms3 / 1e6}
        # config 4 (one-GPU reference): VARCOEF8 fp64 768^3, 8 grids read, 20 sweeps, check every 10
        try:
            n4 = 768
            a4 = gscl.Grid(n4, n4, n4, 1).fill_random(SEED, 0)
            b4 = gscl.Grid(n4, n4, n4, 1)
            cs4 = [gscl.Grid(n4, n4, n4, 0).fill_random(SEED, 2 + i, 0.125) for i in range(7)]
            ms4 = timed(lambda: gscl.jacobi_run("VARCOEF8", a4, b4, iters=20, check_every=10, coeffs=cs4), 2)
            sum4 = gscl.do_reduce("VALUE", [a4], "SUM")  # the final SUM of u
            p4 = float(n4) ** 3 * 20
            # two sweeps per pass (sweep2v): u + 7 coefficients read and v written
            # once per two point-updates = 36 B per point-sweep
            others["config4_varcoef8_768cubed_1gpu"] = {"ms_per_step": ms4, "Gpts": p4 / ms4 / 1e6,
                                                        "hbm_gbs_algorithmic": 36.0 * p4 / ms4 / 1e6,
                                                        "single_sweep_equiv_gbs": 72.0 * p4 / ms4 / 1e6,
                                                        "final_sum_u": sum4}
            for g in [a4, b4] + cs4:
                g.destroy()
        except Exception as ex:
            others["config4_varcoef8_768cubed_1gpu"] = {"error": str(ex)[:200]}
        torch.cuda.empty_cache()

    # ---- end to end: public API with host buffers.  Every step uploads its input
    # grid from pinned host memory (gscl_grid_copy_from_host_async: contiguous H2D
    # + on-device repack on the library's copy stream) and reads its residual
    # history back; two grid sets pipeline step k+1's upload under step k's sweeps.
    gscl.set_option("transport", 0 if not one_gpu else 1)  # (the peer set is bound to u / v)
    host = torch.empty(u.dense_shape(), dtype=torch.float64, pin_memory=True).numpy()
    u.to_host(host)
    u2 = gscl.Grid(n, n, nz, 1) if not one_gpu else u
    v2 = gscl.Grid(n, n, nz, 1) if not one_gpu else v
    sets = [(u, v), (u2, v2)]
    e2e_steps = max(2, args.steps)
    if not one_gpu:  # warm-up: the two upload staging slots are allocated on first use
        u.from_host_async(host)
        u2.from_host_async(host)
        gscl.sync()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sets[0][0].from_host_async(host)
    for k in range(e2e_steps):
        if k + 1 < e2e_steps and not one_gpu:
            sets[(k + 1) % 2][0].from_host_async(host)
        elif one_gpu and k > 0:
            u.from_host(host)  # (one grid set: upload, then run)
        hist = gscl.jacobi_run("JACOBI7", sets[k % 2][0], sets[k % 2][1], iters=iters, check_every=check)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks([time.perf_counter() - t0])[0]
    e2e_val = pts_step / (e2e_s / e2e_steps) / 1e9
    # the same with the final iterate copied back to host memory every step
    # (the paper's context copies the data back at GSCL_End, PAPER.md:85-95,
    # 133): step k's result downloads (gscl_grid_copy_to_host_async, its own
    # stream) while step k+1 uploads and runs on the other grid set
    outs = [torch.empty(u.dense_shape(), dtype=torch.float64, pin_memory=True).numpy() for _ in range(2)]
    fin_steps = e2e_steps
    u.to_host_async(outs[0])  # warm-up: the two download staging slots
    u.to_host_async(outs[1])
    gscl.sync()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if not one_gpu:
        sets[0][0].from_host_async(host)
    for k in range(fin_steps):
        if one_gpu:
            u.from_host(host)
        elif k + 1 < fin_steps:
            sets[(k + 1) % 2][0].from_host_async(host)
        gu, gv = sets[k % 2]
        gscl.jacobi_run("JACOBI7", gu, gv, iters=iters, check_every=check)
        gu.to_host_async(outs[k % 2])
        if one_gpu:
            gscl.sync()
    gscl.sync()
    fin_s = max_over_ranks([time.perf_counter() - t0])[0]
    fin_val = pts_step / (fin_s / fin_steps) / 1e9
    outh = outs[0]
    if not one_gpu:
        u2.destroy()
        v2.destroy()

    # ---- N > 1: the peer-memory transport beside the NCCL headline, measured
    # last (a failure must not cost the NCCL numbers).  Every rank runs the
    # same sequence of host collectives whatever fails locally, and all ranks
    # agree on success before each stage, so a failing rank cannot leave the
    # others waiting in a gloo collective.
    if world > 1 and (not one_gpu or args.p2p_leg) and not args.no_p2p:
        def agree(ok):
            return max_over_ranks([0.0 if ok else 1.0])[0] == 0.0

        def p2p_leg():
            err = None
            blob = None
            try:
                blob = gscl.peer_export(u, v)
            except Exception as ex:
                err = f"peer_export: {ex}"
            blobs = gather(blob)
            ok = err is None and all(b is not None for b in blobs)
            if ok:
                try:
                    gscl.peer_import(u, v, blobs)
                    gscl.set_option("transport", 1)
                except Exception as ex:
                    ok, err = False, f"peer_import: {ex}"
            if not agree(ok):
                return {"error": (err or "peer setup failed on another rank")[:300]}
            nst = max(2, min(args.steps, 5))
            el = None
            barrier()
            try:
                for _ in range(2):
                    step()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(nst):
                    step()
                e1.record(stream)
                torch.cuda.synchronize()
                el = e0.elapsed_time(e1) / nst
            except Exception as ex:
                err = f"step: {ex}"
            if not agree(el is not None):
                return {"error": (err or "a step failed on another rank")[:300]}
            tp = max_over_ranks([el])[0]
            xe = None
            barrier()
            try:
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                gscl.halo_exchange_depth([u], 2)
                torch.cuda.synchronize()
                a0.record(stream)
                for _ in range(50):
                    gscl.halo_exchange_depth([u], 2)
                a1.record(stream)
                torch.cuda.synchronize()
                xe = a0.elapsed_time(a1) / 50
            except Exception as ex:
                err = f"exchange: {ex}"
            if not agree(xe is not None):
                return {"error": (err or "the exchange failed on another rank")[:300]}
            xe = max_over_ranks([xe])[0]
            t_comp = halo["compute_only_ms_per_step"]
            res = {"step_ms": tp, "value": pts_step / (tp * 1e-3) / 1e9, "unit": UNIT,
                   "exchange_only_ms": {"depth2": xe},
                   "exposed_ms_per_step": tp - t_comp, "exposed_ms_per_pass": (tp - t_comp) / (iters // 2),
                   "how": "boundary planes stored into the neighbours by the pass kernel (IPC / NVLink peer "
                          "memory), counter waits"}
            dg, hh = None, None
            try:
                u.fill_random(SEED, 0)
                hh = step()
                dg = u.digest()
            except Exception as ex:
                err = f"parity step: {ex}"
            if agree(dg is not None) and rank == 0 and parity_ref is not None:
                rel = max((abs(a - b) / max(abs(b), 1e-300) for a, b in zip(hh, parity_ref["hist"])), default=0.0)
                res["parity"] = {"ok": dg == parity_ref["digest"] and rel <= 1e-10, "digest": f"{dg:016x}",
                                 "hist_max_rel": rel}
            return res

        halo["p2p_leg" if one_gpu else "p2p"] = leg = p2p_leg()
        halo["p2p"] = halo.get("p2p", leg)
        if parity is not None and rank == 0 and "parity" in leg:
            parity["p2p_leg" if one_gpu else "p2p"] = pl = leg.pop("parity")
            parity["parity_ok"] = bool(parity.get("parity_ok")) and pl["ok"]

    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            os.sched_setaffinity(0, all_cpus)  # the oracle gets every host core
            base = cpu_baseline(min(n, 512))
        except Exception as ex:  # the baseline must not sink the GPU number
            base = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle",
                    "sample": f"failed: {ex}"}
    if rank == 0:
        grid_bytes = 2 * u.nbytes
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step,
            "ms_per_step_median": statistics.median(per_step), "ms_per_step_min": min(per_step),
            "ms_per_step_max": max(per_step),
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (splitmix64 U[0,1) interior, zero Dirichlet halo; state carried across steps)",
            "config": {
                "workload": (f"config2: JACOBI7 fp64 {n}^3 + halo 1, {iters} sweeps, L2 residual fused "
                             f"every {check} + final" + (" (two sweeps per HBM pass)" if n_k[3] > 0 else "")
                             if world == 1 else
                             f"config5: weak scaling JACOBI7 fp64 {n}^3 per GPU (global {n}x{n}x{nz}), "
                             f"{iters} sweeps, z-halo exchange ({transport}), residual every {check}"),
                "global_grid": [n, n, nz], "sweeps_per_step": iters, "check_every": check,
                "parallelism": f"zslab{world}",
                "l2": (f"inputs larger than L2 (2 x {u.nbytes / 1e9:.2f} GB per GPU vs 126 MB), no flush"
                       if grid_bytes > L2_BYTES else
                       f"inputs fit in L2 (2 x {u.nbytes / 1e6:.1f} MB per GPU vs 126 MB): not an HBM number"),
                "halo_transport": transport,
                "sweep_equiv_gbs": value * BYTES_PER_PT / world,
                "sweep_equiv_gbs_note": "per GPU, 16 B per point-update as if every sweep streamed HBM; "
                                        "the two-sweep pass moves half of that (roofline.achieved is HBM)",
            },
            "roofline": roof,
            "cpu_baseline": base,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(host.nbytes),
                    "d2h_bytes_per_step": 8 * len(hist), "steps": e2e_steps,
                    "host_cpus": numa_cpus,
                    "how": "per step: pinned-host upload of the input grid (async, copy stream, "
                           "double-buffered) + jacobi_run + residual history read back; wall clock",
                    "with_final_iterate": {"value": fin_val, "unit": UNIT, "h2d_bytes_per_step": int(host.nbytes),
                                           "d2h_bytes_per_step": int(outh.nbytes) + 8 * len(hist),
                                           "steps": fin_steps,
                                           "how": "per step: pinned-host upload (async, copy stream), jacobi_run, "
                                                  "the final iterate copied back to pinned host memory "
                                                  "(gscl_grid_copy_to_host_async, download stream); two grid "
                                                  "sets, so step k's download overlaps step k+1's upload and "
                                                  "sweeps; all downloads landed (gscl_sync) before the clock "
                                                  "stops; wall clock"}},
            "gpu_launches": int(launches),
            "single_sweep_schedule": single,
            "other_configs": others,
            "clocks": clk.summary(),
            "residual_last": hist[-1] if hist else None,
        }
        if halo is not None:
            line["halo"] = halo
        if parity is not None:
            line["parity"] = parity
        print(json.dumps(line), flush=True)
    try:
        gscl.finalize()
    except Exception:
        pass
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gscl", choices=["gscl", "reference"])
    ap.add_argument("--n", "--size", dest="n", type=int, default=512)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--check-every", type=int, default=10)
    ap.add_argument("--ref-iters", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next2", "--no-single-sweep", dest="no_next2", action="store_true",
                    help="skip the one-sweep-per-pass comparison run")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-p2p", action="store_true", help="N > 1: skip the peer-memory transport leg")
    ap.add_argument("--no-parity", action="store_true", help="N > 1: skip the single-domain check")
    ap.add_argument("--p2p-leg", action="store_true",
                    help="with --one-gpu-ranks: also run the separate peer-transport leg (testing)")
    ap.add_argument("--timeout-ms", type=int, default=60000, help="N > 1: the library's watchdog")
    ap.add_argument("--single-domain", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--clock-ms", type=int, default=20, help="nvidia-smi clock sampling period in the timed region")
    ap.add_argument("--one-gpu-ranks", action="store_true",
                    help="debug: run every torchrun rank on GPU 0 (gloo + peer transport, no NCCL); "
                         "exercises the multi-rank path on a one-GPU box, numbers are meaningless")
    args = ap.parse_args()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.warmup < 3:
        args.warmup = 3
    if args.single_domain:
        run_single_domain(args)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_gpu(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
