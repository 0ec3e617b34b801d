cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
for o in zchunks=0 zchunks=8 zchunks=12 zchunks=6 zchunks=4 zchunks=0 zchunks=8; do timeout 300 python tools/jacobi_probe.py --op JACOBI27 --steps 3 --opts $o 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); k=d['kernel_ms']; n=d['launches']; print(d['opts'], round(d['Gpts'],1), 'sweep', round(k[0]/max(n[0],1),4), 'fused', round(k[1]/max(n[1],1),4), 'resid', round(k[2]/max(n[2],1),4))"; done
for o in zchunks=0 zchunks=32 zchunks=16; do timeout 300 python tools/jacobi_probe.py --steps 3 --opts tblock=1,$o 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); k=d['kernel_ms']; n=d['launches']; print('J7', d['opts'], round(d['Gpts'],1), 'sweep', round(k[0]/max(n[0],1),4), 'fused', round(k[1]/max(n[1],1),4), 'resid', round(k[2]/max(n[2],1),4))"; done
