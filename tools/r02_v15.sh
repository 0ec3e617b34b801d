# 8 consumer warps + producer warpgroup (variant 15) vs the default, with out-of-grid warps idle
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
timeout 300 python tools/variant_digest.py 15 > gpurun_out/v15_digest.log 2>&1
O=gpurun_out/v15_ab.jsonl; : > $O
for rep in 1 2 3; do
  timeout 300 python tools/jacobi_probe.py --steps 5 --opts variant=0 variant=15 >> $O
done
tail -3 gpurun_out/v15_digest.log
