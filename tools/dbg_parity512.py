"""Diagnose full-size parity: where (plane/row/col) does the GPU differ from the oracle."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
import oracle
from paper_1207_1746_b200 import gscl

SEED = 12071746


def report(tag, got, ref):
    d = got.view(np.uint64) != ref.view(np.uint64)
    n = int(d.sum())
    print(tag, "diff cells:", n, flush=True)
    if n:
        idx = np.argwhere(d)
        pl = np.unique(idx[:, 0]); rw = np.unique(idx[:, 1]); cl = np.unique(idx[:, 2])
        print("  planes", pl[:10], "...", pl[-5:], len(pl))
        print("  rows", rw[:10], "...", rw[-5:], len(rw))
        print("  cols", cl[:10], "...", cl[-5:], len(cl))
        i = tuple(idx[0]); print("  first", i, got[i], ref[i])


def main():
    gscl.init(0, 1, device=0)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    for iters in [1, 2, 3, 10]:
        u = gscl.Grid(n, n, n, 1).fill_random(SEED, 0)
        v = gscl.Grid(n, n, n, 1)
        hist = gscl.jacobi_run("JACOBI7", u, v, iters=iters, check_every=0)
        got = u.to_host()
        a = oracle.alloc(n, n, n, 1); oracle.fill_random(a, 1, SEED, 0)
        fin, _ = oracle.jacobi_run("JACOBI7", a, oracle.alloc(n, n, n, 1), 1, iters, 0)
        report(f"jacobi iters={iters}", got, fin)
        print("  digest gpu", u.digest(), "oracle", oracle.digest(fin, 1), "host", oracle.digest(got, 1))
        u.destroy(); v.destroy()


main()
