timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "test_jacobi_temporal_blocking" > gpurun_out/g3_pytest.log 2>&1; tail -3 gpurun_out/g3_pytest.log
for v in 0 50 51 52 53 54 40 0; do timeout 300 python tools/jacobi_probe.py --opts variant=$v --steps 5 2>&1 | tail -1; done | tee gpurun_out/g3_probe.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['opts'], round(d['Gpts'],1), 'pass_ms', round(d['kernel_ms'][3]/d['launches'][3],4))"
