#!/bin/bash
# ncu evidence for the bench step: the launch list of `bench.py --steps 1 --warmup 3`
# (cold-cache, serialised; compare shares) and one --set full capture of the
# two-sweep pass and of the do_all sweep.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-configs \
    --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep2r_tma -s 4 -c 1 \
    -o gpurun_out/pass_full python tools/jacobi_probe.py --iters 10 --check 0 --steps 1 --no-timing \
    > gpurun_out/pass_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_tma -s 4 -c 1 \
    -o gpurun_out/sweep_full python tools/jacobi_probe.py --iters 10 --check 0 --steps 1 --no-timing \
    --opts tblock=1 > gpurun_out/sweep_full.log 2>&1
ls -la gpurun_out
