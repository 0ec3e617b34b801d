cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --one-gpu-ranks --size 128 --steps 3 > gpurun_out/gB_bench_n2.jsonl 2> gpurun_out/gB_bench_n2.err; echo "n2 rc=$?"; tail -c 2500 gpurun_out/gB_bench_n2.jsonl; tail -5 gpurun_out/gB_bench_n2.err
timeout 900 python bench.py > gpurun_out/gB_bench.jsonl 2> gpurun_out/gB_bench.err; echo "n1 rc=$?"; tail -c 4000 gpurun_out/gB_bench.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gB_pytest.log 2>&1; tail -3 gpurun_out/gB_pytest.log
