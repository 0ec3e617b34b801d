cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for lib in libgscl_base.so libgscl.so libgscl_base.so libgscl.so; do
  GSCL_LIB=paper_1207_1746_b200/$lib timeout 300 python tools/jacobi_probe.py --steps 5 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); k=d['kernel_ms']; n=d['launches']; print('$lib', round(d['Gpts'],1), 'pass', round(k[3]/max(n[3],1),4))"
  GSCL_LIB=paper_1207_1746_b200/$lib timeout 300 python tools/jacobi_probe.py --steps 5 --check 0 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); k=d['kernel_ms']; n=d['launches']; print('$lib nocheck', round(d['Gpts'],1), 'pass', round(k[3]/max(n[3],1),4))"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "jacobi or split or pass2 or rbgs or converge" 2>&1 | tail -2
