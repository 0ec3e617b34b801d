# 27-point reduction sweeps with 6 consumer warps (no 128-register spills) vs 7
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "27 or reduce or fused or jacobi" > gpurun_out/k6_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k6_pytest.log
O=gpurun_out/k6_ab.jsonl; : > $O
for rep in 1 2 3; do
for lib in libgscl_prev.so libgscl.so; do
  GSCL_LIB=paper_1207_1746_b200/$lib timeout 300 python tools/jacobi_probe.py --op JACOBI27 --steps 3 | sed "s/^/{\"lib\": \"$lib\", \"rec\": /; s/\$/}/" >> $O
done; done
tail -2 gpurun_out/k6_pytest.log
