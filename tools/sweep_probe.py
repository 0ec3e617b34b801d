"""Per-kernel timing probe (not the bench): CUDA-event time per launch of the
sweep kernels at full size, for tuning and ablations.  Prints JSON lines."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ops", default="JACOBI7,JACOBI27,FIG1B,VARCOEF8")
    ap.add_argument("--impls", default="0,1")
    ap.add_argument("--zchunks", default="0")
    ap.add_argument("--vn", type=int, default=384, help="VARCOEF8 edge (memory)")
    ap.add_argument("--copy", action="store_true")
    ap.add_argument("--dtype", type=int, default=0)
    ap.add_argument("--l2promo", default="0")
    ap.add_argument("--sched", default="0")
    ap.add_argument("--stages", default="0")
    ap.add_argument("--variant", default="0")
    args = ap.parse_args()
    import torch
    from paper_1207_1746_b200 import gscl
    gscl.init(0, 1, device=0)
    if args.copy:
        a = torch.empty(2**27, dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        for _ in range(3):
            b.copy_(a)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(args.reps):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        print(json.dumps({"kernel": "torch_copy_1GiB_f64", "ms": ms, "GBps": 2 * a.numel() * 8 / ms / 1e6}))
        del a, b
    for op in args.ops.split(","):
        n = args.vn if op == "VARCOEF8" else args.n
        es = 8 if args.dtype == 0 else 4
        u = gscl.Grid(n, n, n, 1, args.dtype).fill_random(12071746, 0)
        v = gscl.Grid(n, n, n, 1, args.dtype)
        ins = [u]
        if op == "VARCOEF8":
            ins += [gscl.Grid(n, n, n, 0, args.dtype).fill_random(12071746, 2 + i, 0.125) for i in range(7)]
        bpp = (2 + (7 if op == "VARCOEF8" else 0)) * es
        import itertools
        combos = itertools.product([int(x) for x in args.impls.split(",")],
                                   [int(x) for x in args.zchunks.split(",")],
                                   [int(x) for x in args.l2promo.split(",")],
                                   [int(x) for x in args.sched.split(",")],
                                   [int(x) for x in args.stages.split(",")],
                                   [int(x) for x in args.variant.split(",")])
        for impl, zc, l2p, sch, stg, var in combos:
            if True:
                gscl.set_option("sweep_impl", impl)
                gscl.set_option("zchunks", zc)
                gscl.set_option("l2promo", l2p)
                gscl.set_option("sched", sch)
                gscl.set_option("stages", stg)
                gscl.set_option("variant", var)
                for _ in range(3):
                    gscl.do_all(op, ins, v)
                gscl.sync()
                gscl.timing_read()
                gscl.timing_enable(True)
                for _ in range(args.reps):
                    gscl.do_all(op, ins, v)
                ms, cnt, _ = gscl.timing_read()
                gscl.timing_enable(False)
                t = ms[0] / cnt[0]
                rec = {"op": op, "n": n, "impl": impl, "zchunks": zc, "l2promo": l2p, "sched": sch, "stages": stg, "variant": var,
                       "dtype": args.dtype, "ms": t,
                       "Gpts": n ** 3 / t / 1e6, "GBps_alg": bpp * n ** 3 / t / 1e6}
                if op in ("JACOBI7", "JACOBI27"):
                    gscl.timing_enable(True)
                    for _ in range(args.reps):
                        gscl.do_reduce(op + "_RESID" + op[-2:].replace("I", "") + "_SQ" if False else
                                       ("JACOBI7_RESID7_SQ" if op == "JACOBI7" else "JACOBI27_RESID27_SQ"),
                                       [u], "SUM", out=v)
                    ms, cnt, _ = gscl.timing_read()
                    gscl.timing_enable(False)
                    rec["fused_ms"] = ms[1] / cnt[1]
                print(json.dumps(rec), flush=True)
        for g in ins + [v]:
            g.destroy()
    gscl.finalize()


if __name__ == "__main__":
    main()
