"""Time gscl_jacobi_run steps (CUDA events on the library stream) under option sets.

  python tools/jacobi_probe.py --op JACOBI7 --n 512 --iters 100 --check 10 --opts split=0 split=1
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="JACOBI7")
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--nz", type=int, default=0)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--check", type=int, default=10)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--dtype", type=int, default=0)
    ap.add_argument("--opts", nargs="*", default=[""])
    ap.add_argument("--no-timing", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_1207_1746_b200 import gscl
    gscl.init(0, 1, device=0)
    n, nz = args.n, args.nz or args.n
    u = gscl.Grid(n, n, nz, 1, args.dtype).fill_random(12071746, 0)
    v = gscl.Grid(n, n, nz, 1, args.dtype)
    cs = []
    if args.op == "VARCOEF8":
        cs = [gscl.Grid(n, n, nz, 0, args.dtype).fill_random(12071746, 2 + i, 0.125) for i in range(7)]
    for optset in args.opts:
        opts = dict(kv.split("=") for kv in optset.split(",") if kv)
        for k, val in opts.items():
            gscl.set_option(k, int(val))
        for _ in range(2):
            gscl.jacobi_run(args.op, u, v, args.iters, args.check, cs)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        gscl.timing_read()
        gscl.timing_enable(not args.no_timing)
        e0.record(st)
        for _ in range(args.steps):
            gscl.jacobi_run(args.op, u, v, args.iters, args.check, cs)
        e1.record(st)
        torch.cuda.synchronize()
        ms_k, n_k, launches = gscl.timing_read()
        gscl.timing_enable(False)
        ms = e0.elapsed_time(e1) / args.steps
        pts = n * n * nz * args.iters
        print(json.dumps({"op": args.op, "n": n, "nz": nz, "dtype": args.dtype, "opts": opts,
                          "ms_per_step": ms, "Gpts": pts / ms / 1e6, "kernel_ms": ms_k, "launches": n_k,
                          "all_launches": launches}), flush=True)
        for k in opts:
            gscl.set_option(k, 0)


if __name__ == "__main__":
    main()
