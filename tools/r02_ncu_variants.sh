# ncu --set full of one two-sweep pass per variant (512^3 fp64), usage: bash tools/r02_ncu_variants.sh TAG v1 v2 ...
tag=$1; shift
for v in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep2r -s 3 -c 1 \
    -o gpurun_out/${tag}_v$v python tools/jacobi_probe.py --opts variant=$v --steps 1 --iters 4 --check 0 > gpurun_out/${tag}_v$v.log 2>&1
  tail -2 gpurun_out/${tag}_v$v.log
done
