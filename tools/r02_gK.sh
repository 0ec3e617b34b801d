# end-of-block validation: full GPU suite (product build), ablation parity subset, sanitizers
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gK_pytest.log 2>&1; tail -3 gpurun_out/gK_pytest.log
GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "temporal_blocking or two_sweep_passes or impl" > gpurun_out/gK_abl.log 2>&1; tail -2 gpurun_out/gK_abl.log
