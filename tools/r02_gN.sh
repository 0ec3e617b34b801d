cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
timeout 120 python tools/variant_digest.py 40 41 42
for v in 0 40 41 42 0 41 42; do timeout 300 python tools/jacobi_probe.py --opts variant=$v --steps 5 --check 0 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['opts'], round(d['Gpts'],1), 'pass_ms', round(d['kernel_ms'][3]/d['launches'][3],4))"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_tma -s 19 -c 1 -o gpurun_out/k27fused python tools/jacobi_probe.py --op JACOBI27 --iters 20 --check 10 --steps 1 --no-timing > gpurun_out/k27fused.log 2>&1; tail -1 gpurun_out/k27fused.log
