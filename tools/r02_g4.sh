# full GPU suite on the product library, ablation parity on the ablation build, then the bench
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/g7_pytest.log 2>&1; tail -3 gpurun_out/g7_pytest.log
GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "temporal_blocking or two_sweep_passes or impl or do_all" > gpurun_out/g7_pytest_abl.log 2>&1; tail -2 gpurun_out/g7_pytest_abl.log
timeout 900 python bench.py > gpurun_out/g7_bench.jsonl 2> gpurun_out/g7_bench.err; tail -c 3000 gpurun_out/g7_bench.jsonl
