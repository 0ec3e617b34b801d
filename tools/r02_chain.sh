# chained two-sweep passes (PDL + per-unit flags): parity suites, A/B, bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_abi_edge.py -m gpu -x -q > gpurun_out/ch_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ch_pytest.log
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
O=gpurun_out/ch_ab.jsonl; : > $O
for rep in 1 2; do
  timeout 300 python tools/jacobi_probe.py --steps 5 --opts chain=0 "" >> $O
  timeout 300 python tools/jacobi_probe.py --steps 5 --no-timing --opts chain=0 "" >> $O
  timeout 300 python tools/jacobi_probe.py --steps 5 --check 0 --opts chain=0 "" >> $O
done
unset GSCL_LIB
timeout 900 python bench.py --no-configs > gpurun_out/ch_bench.jsonl 2> gpurun_out/ch_bench.err
tail -2 gpurun_out/ch_pytest.log
