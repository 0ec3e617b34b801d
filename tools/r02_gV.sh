cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
timeout 120 python tools/variant_digest.py 44 45
for v in 0 44 45 0 44 45; do timeout 300 python tools/jacobi_probe.py --opts variant=$v --steps 5 --check 0 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('nocheck', d['opts'], round(d['Gpts'],1), 'pass_ms', round(d['kernel_ms'][3]/d['launches'][3],4))"; done
