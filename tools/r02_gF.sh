cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
pr() { python -c "
import sys,json
l=[x for x in sys.stdin if x.startswith('{')][-1]; d=json.loads(l); r=d['roofline']
print(round(d['value'],1), 'pass', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), d['clocks'].get('source'))"; }
timeout 300 python tools/jacobi_probe.py --steps 5 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('probe', round(d['Gpts'],1), 'pass_ms', round(d['kernel_ms'][3]/d['launches'][3],4))"
for ms in 20 1000 20 1000; do timeout 600 python bench.py --no-cpu-baseline --no-configs --no-next2 --clock-ms $ms 2>/dev/null | pr; done
timeout 300 python tools/jacobi_probe.py --steps 5 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('probe', round(d['Gpts'],1), 'pass_ms', round(d['kernel_ms'][3]/d['launches'][3],4))"
