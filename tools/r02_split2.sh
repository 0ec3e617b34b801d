# boundary chunks and middle chunks of the multi-rank JACOBI7 pass as two launches
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_peer_multiproc.py tests/test_gpu_abi_edge.py -m gpu -x -q > gpurun_out/s2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2_pytest.log
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
O=gpurun_out/s2_ab.jsonl; : > $O
for rep in 1 2; do
  timeout 300 python tools/jacobi_probe.py --steps 5 --opts "" split=1 split=1,split_one=1 >> $O
  timeout 300 python tools/jacobi_probe.py --steps 5 --check 0 --opts "" split=1 split=1,split_one=1 >> $O
done
unset GSCL_LIB
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --one-gpu-ranks --size 128 --steps 3 > gpurun_out/s2_bench_n2.jsonl 2> gpurun_out/s2_bench_n2.err
tail -2 gpurun_out/s2_pytest.log
