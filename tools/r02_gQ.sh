cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python tools/mr_probe.py
for o in "" split=1 "" split=1; do timeout 300 python tools/jacobi_probe.py --steps 5 --opts "$o" 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); k=d['kernel_ms']; n=d['launches']; print(d['opts'], round(d['Gpts'],1), 'pass', round(k[3]/max(n[3],1),4))"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split or pass2 or peer or converge" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_peer_multiproc.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "multirank" 2>&1 | tail -2
