# round-2 final validation (sixth pass: rows fetched straight into the tuple registers)
# multi-rank bench path on one GPU, ncu launch list of the bench step and --set full captures
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/fin6_gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/fin6_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin6_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin6_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin6_smoke.log
timeout 900 python bench.py > gpurun_out/fin6_bench.jsonl 2> gpurun_out/fin6_bench.err; echo "bench rc=$?" >> gpurun_out/fin6_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/fin6_bench_ref.jsonl 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --one-gpu-ranks --size 128 --steps 3 > gpurun_out/fin6_bench_n2_onegpu.jsonl 2> gpurun_out/fin6_bench_n2_onegpu.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/fin6_launches.csv python bench.py --steps 1 --warmup 3 --no-configs --no-cpu-baseline --no-next2 > gpurun_out/fin6_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep2r_tma -s 4 -c 1 -o gpurun_out/fin6_pass python tools/jacobi_probe.py --iters 10 --check 0 --steps 1 --no-timing > /dev/null 2>&1

ncu --set full --clock-control none --import-source on -k regex:sweep2r_tma -s 20 -c 2 -o gpurun_out/fin6_split python tools/jacobi_probe.py --iters 10 --check 0 --steps 1 --no-timing --opts split=1 > /dev/null 2>&1
tail -2 gpurun_out/fin6_pytest.log; tail -1 gpurun_out/fin6_smoke.log; tail -1 gpurun_out/fin6_bench.err; ls gpurun_out | grep fin6_
