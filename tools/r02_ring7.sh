# 7-warp do_all: 4 (default) / 6 / 5-stage rings at 3 CTAs per SM (variants 57 / 58)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
O=gpurun_out/ring7_ab.jsonl; : > $O
for rep in 1 2 3; do
  timeout 300 python tools/jacobi_probe.py --steps 3 --opts tblock=1,variant=0 tblock=1,variant=57 tblock=1,variant=58 >> $O
done
