# do_all JACOBI7 with one row per lane (variant 57: 7 consumer warps, 3 CTAs per SM) vs the default (2 rows, 3 CTAs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
O=gpurun_out/nw7_ab.jsonl; : > $O
for rep in 1 2 3; do
  timeout 300 python tools/jacobi_probe.py --steps 3 --opts tblock=1,variant=0 tblock=1,variant=57  >> $O
done
N=257 timeout 300 python - > gpurun_out/nw7_digest.log 2>&1 <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1207_1746_b200 import gscl
gscl.init(0, 1, device=0)
n = 257
res = {}
for v in (0, 57):
    gscl.set_option("tblock", 1)
    gscl.set_option("variant", v)
    u = gscl.Grid(n, n - 3, n - 5, 1).fill_random(12071746, 0)
    w = gscl.Grid(n, n - 3, n - 5, 1)
    gscl.jacobi_run("JACOBI7", u, w, iters=21, check_every=0)
    res[v] = u.digest()
    u.destroy(); w.destroy()
print({k: (hex(d), d == res[0]) for k, d in res.items()})
PY
cat gpurun_out/nw7_digest.log
