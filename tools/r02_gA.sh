# ADVICE fixes: peer transport (slot counters, final wait, watchdog), NULL stream graphs, halo-plane memcmp
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer_multiproc.py tests/test_gpu_abi_edge.py -x -q > gpurun_out/gA_pytest.log 2>&1; tail -15 gpurun_out/gA_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "jacobi or converge or rbgs" > gpurun_out/gA_parity.log 2>&1; tail -3 gpurun_out/gA_parity.log
