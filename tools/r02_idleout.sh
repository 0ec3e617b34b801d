# idle out-of-grid warps skip the ring: parity + A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_abi_edge.py -m gpu -x -q > gpurun_out/io_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/io_pytest.log
O=gpurun_out/io_ab.jsonl; : > $O
for rep in 1 2 3; do
for lib in libgscl_prev.so libgscl.so; do
  GSCL_LIB=paper_1207_1746_b200/$lib timeout 300 python tools/jacobi_probe.py --steps 10 --no-timing | sed "s/^/{\"lib\": \"$lib\", \"rec\": /; s/\$/}/" >> $O
done; done
tail -2 gpurun_out/io_pytest.log
