# A/B: streaming (evict-first) output stores vs default stores
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for lib in libgscl_base.so libgscl.so libgscl_base.so libgscl.so; do
  echo "== $lib"
  GSCL_LIB=paper_1207_1746_b200/$lib timeout 300 python tools/jacobi_probe.py --steps 5 --opts "" tblock=1 2>&1 | tail -2 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); k=d['kernel_ms']; n=d['launches']; print(d['opts'], round(d['Gpts'],1), 'sweep', round(k[0]/max(n[0],1),4), 'pass', round(k[3]/max(n[3],1),4))"
  GSCL_LIB=paper_1207_1746_b200/$lib timeout 300 python tools/jacobi_probe.py --op VARCOEF8 --n 768 --iters 20 --check 10 --steps 3 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); k=d['kernel_ms']; n=d['launches']; print('v8', round(d['Gpts'],1), 'pass', round(k[3]/max(n[3],1),4))"
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:sweep_tma -s 6 -c 2 python tools/jacobi_probe.py --steps 1 --iters 10 --check 0 --opts tblock=1 2>&1 | grep -E "dram__|duration" | head -6
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:sweep2r -s 6 -c 2 python tools/jacobi_probe.py --steps 1 --iters 10 --check 0 2>&1 | grep -E "dram__|duration" | head -6
