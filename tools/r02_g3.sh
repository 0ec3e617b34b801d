for v in 0 94 95 96 97 98 99 0 94; do timeout 300 python tools/jacobi_probe.py --opts variant=$v --steps 5 2>&1 | tail -1; done | tee gpurun_out/g6_probe.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['opts'], round(d['Gpts'],1), 'pass_ms', round(d['kernel_ms'][3]/d['launches'][3],4))"
