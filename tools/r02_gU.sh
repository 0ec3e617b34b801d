cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
timeout 120 python tools/variant_digest.py 98
for v in 0 98 0 98; do timeout 300 python tools/jacobi_probe.py --opts variant=$v --steps 5 --check 0 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('nocheck', d['opts'], round(d['Gpts'],1), 'pass_ms', round(d['kernel_ms'][3]/d['launches'][3],4))"; done
for v in 0 98; do timeout 300 python tools/jacobi_probe.py --opts variant=$v --steps 5 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['opts'], round(d['Gpts'],1), 'pass_ms', round(d['kernel_ms'][3]/d['launches'][3],4))"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep2r -s 3 -c 1 -o gpurun_out/dyn98b python tools/jacobi_probe.py --opts variant=98 --steps 1 --iters 4 --check 0 > /dev/null 2>&1; ls gpurun_out | grep dyn98b
