# where do the ring waits go with a continuous ring (variant 98, persistent CTAs)?
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GSCL_LIB=paper_1207_1746_b200/libgscl_ablations.so
for v in 0 98; do
ncu --set full --clock-control none --import-source on -k regex:sweep2r_tma -s 4 -c 1 -o gpurun_out/dyn_v$v python tools/jacobi_probe.py --iters 10 --check 0 --steps 1 --no-timing --opts variant=$v > gpurun_out/dyn_v$v.log 2>&1
done
ls gpurun_out | grep dyn_
