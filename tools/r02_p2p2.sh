# peer transport with the two-launch JACOBI7 pass: multi-process peer tests, parity, bench n2 on one GPU
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_peer_multiproc.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/p2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p2_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --one-gpu-ranks --size 128 --steps 3 > gpurun_out/p2_bench_n2.jsonl 2> gpurun_out/p2_bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 3 --one-gpu-ranks --size 128 --steps 3 > gpurun_out/p2_bench_n3.jsonl 2> gpurun_out/p2_bench_n3.err
tail -2 gpurun_out/p2_pytest.log
