# z-chunk count of the final pass (ablation knob zchunks; auto = 6 at 512^3)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
O=gpurun_out/zch_ab.jsonl; : > $O
for rep in 1 2; do
  timeout 600 python tools/jacobi_probe.py --steps 5 --opts zchunks=0 zchunks=4 zchunks=5 zchunks=7 zchunks=8 >> $O
done
