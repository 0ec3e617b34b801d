# run-level pass timing and the faster copy_halo: parity, probe with / without timing, bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_abi_edge.py -m gpu -x -q > gpurun_out/tm_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tm_pytest.log
O=gpurun_out/tm_ab.jsonl; : > $O
for rep in 1 2; do
  timeout 300 python tools/jacobi_probe.py --steps 5 >> $O
  timeout 300 python tools/jacobi_probe.py --steps 5 --no-timing >> $O
done
timeout 900 python bench.py > gpurun_out/tm_bench.jsonl 2> gpurun_out/tm_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_copy_halo -c 4 --csv python tools/jacobi_probe.py --iters 10 --check 0 --steps 1 --no-timing > gpurun_out/tm_copyhalo.csv 2>&1
tail -2 gpurun_out/tm_pytest.log
