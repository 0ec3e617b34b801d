set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "test_jacobi_temporal_blocking" 2>&1 | tail -5
for v in 0 40 42 43 46 48 49 0; do timeout 300 python tools/jacobi_probe.py --opts variant=$v --steps 5 2>&1 | tail -1; done | tee gpurun_out/g1_probe.jsonl
