# VARCOEF8 multi-rank pass as boundary + middle launches
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_peer_multiproc.py tests/test_gpu_abi_edge.py -m gpu -x -q > gpurun_out/s2v_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2v_pytest.log
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
O=gpurun_out/s2v_ab.jsonl; : > $O
for rep in 1 2; do
  timeout 600 python tools/jacobi_probe.py --op VARCOEF8 --n 768 --steps 2 --opts "" split=1 split=1,split_one=1 >> $O
done
tail -2 gpurun_out/s2v_pytest.log
