# PROBE: longer leading z-chunks so the last wave's units (the last chunk) are shorter
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
O=gpurun_out/chadd_ab.jsonl; : > $O
for rep in 1 2; do
for add in 0 2 4 6; do
  GSCL_PASS_CHUNK_ADD=$add timeout 300 python tools/jacobi_probe.py --steps 5 | sed "s/^/{\"add\": $add, \"rec\": /; s/\$/}/" >> $O
done; done
