# RESID7^2 fold in the two-sweep pass: FMA (+ fast-path without select) vs the two-rounding form
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/fma_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fma_pytest.log
O=gpurun_out/fma_ab.jsonl; : > $O
for rep in 1 2 3; do
for lib in libgscl_base.so libgscl_fmasel.so libgscl_fmafast.so; do
  GSCL_LIB=paper_1207_1746_b200/$lib timeout 300 python tools/jacobi_probe.py --steps 5 | sed "s/^/{\"lib\": \"$lib\", \"rec\": /; s/\$/}/" >> $O
done; done
tail -2 gpurun_out/fma_pytest.log
