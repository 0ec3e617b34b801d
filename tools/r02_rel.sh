# A/B: stage release by data dependency (new) vs fence.proxy.async (prev build)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
O=gpurun_out/rel_ab.jsonl; : > $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/rel_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rel_pytest.log
for rep in 1 2; do
for lib in libgscl_prev.so libgscl.so; do
  export GSCL_LIB=paper_1207_1746_b200/$lib
  timeout 300 python tools/jacobi_probe.py --steps 5 | sed "s/^/{\"lib\": \"$lib\", \"rec\": /; s/\$/}/" >> $O
  timeout 300 python tools/jacobi_probe.py --steps 5 --check 0 | sed "s/^/{\"lib\": \"$lib\", \"rec\": /; s/\$/}/" >> $O
  timeout 300 python tools/jacobi_probe.py --steps 3 --opts tblock=1 | sed "s/^/{\"lib\": \"$lib\", \"rec\": /; s/\$/}/" >> $O
  timeout 300 python tools/jacobi_probe.py --op JACOBI27 --steps 3 | sed "s/^/{\"lib\": \"$lib\", \"rec\": /; s/\$/}/" >> $O
  timeout 300 python tools/jacobi_probe.py --op VARCOEF8 --n 768 --steps 2 | sed "s/^/{\"lib\": \"$lib\", \"rec\": /; s/\$/}/" >> $O
done
done
unset GSCL_LIB
tail -2 gpurun_out/rel_pytest.log
