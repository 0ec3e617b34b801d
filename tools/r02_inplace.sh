# rows fetched straight into the tuple c fields (no register copies): parity + A/B vs previous build
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_peer_multiproc.py -m gpu -x -q > gpurun_out/ip_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ip_pytest.log
O=gpurun_out/ip_ab.jsonl; : > $O
for rep in 1 2 3; do
for lib in libgscl_prev.so libgscl.so; do
  GSCL_LIB=paper_1207_1746_b200/$lib timeout 300 python tools/jacobi_probe.py --steps 5 | sed "s/^/{\"lib\": \"$lib\", \"rec\": /; s/\$/}/" >> $O
done; done
tail -2 gpurun_out/ip_pytest.log
