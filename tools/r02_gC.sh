cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "varcoef8 or pass2 or split" > gpurun_out/gC_parity.log 2>&1; tail -3 gpurun_out/gC_parity.log
timeout 900 python -m pytest tests/test_gpu_peer_multiproc.py -x -q > gpurun_out/gC_peer.log 2>&1; tail -3 gpurun_out/gC_peer.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --one-gpu-ranks --size 128 --steps 3 > gpurun_out/gC_bench_n2.jsonl 2> gpurun_out/gC_bench_n2.err; echo "n2 rc=$?"
python - <<'PY'
import json
l=[x for x in open("gpurun_out/gC_bench_n2.jsonl") if x.startswith("{")][-1]
d=json.loads(l); print(json.dumps(d.get("parity")), json.dumps(d.get("halo"))[:600])
PY
timeout 300 python tools/jacobi_probe.py --op VARCOEF8 --n 768 --iters 20 --check 10 --steps 3 --opts "" split=1 2>&1 | tail -2
