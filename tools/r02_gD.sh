# A/B: 27-point sweeps with 7 consumer warps (128 registers, no spills) vs 8 (96, spills)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
for lib in libgscl_base.so libgscl.so libgscl_base.so libgscl.so; do
  echo "== $lib"; GSCL_LIB=paper_1207_1746_b200/$lib timeout 300 python tools/jacobi_probe.py --op JACOBI27 --steps 3 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(round(d['Gpts'],1), 'ms', round(d['ms_per_step'],2), 'sweep', round(d['kernel_ms'][0]/max(d['launches'][0],1),4), 'fused', round(d['kernel_ms'][1]/max(d['launches'][1],1),4), 'resid', round(d['kernel_ms'][2]/max(d['launches'][2],1),4))"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "27" 2>&1 | tail -2
ncu --set full --clock-control none --import-source on -k regex:sweep_tma -s 12 -c 2 -o gpurun_out/k27_r02 python tools/jacobi_probe.py --op JACOBI27 --iters 20 --check 10 --steps 1 --no-timing > gpurun_out/k27_r02.log 2>&1; tail -2 gpurun_out/k27_r02.log
