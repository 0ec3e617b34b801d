# ring stages released in pairs / quads (variants 88 / 89) vs one per plane
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
timeout 300 python tools/variant_digest.py 88 89 > gpurun_out/rel2_digest.log 2>&1
O=gpurun_out/rel2_ab.jsonl; : > $O
for rep in 1 2 3; do
  timeout 300 python tools/jacobi_probe.py --steps 5 --opts variant=0 variant=88 variant=89 >> $O
done
cat gpurun_out/rel2_digest.log | tail -5
