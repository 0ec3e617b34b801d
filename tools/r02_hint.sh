# consumer ring wait with a suspend-time hint (500 / 2000 ns) vs plain try_wait polling
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
GSCL_LIB=paper_1207_1746_b200/libgscl_h500.so timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "jacobi or pass" > gpurun_out/hint_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/hint_pytest.log
O=gpurun_out/hint_ab.jsonl; : > $O
for rep in 1 2 3; do
for lib in libgscl_prev.so libgscl_h500.so libgscl_h2000.so; do
  GSCL_LIB=paper_1207_1746_b200/$lib timeout 300 python tools/jacobi_probe.py --steps 5 | sed "s/^/{\"lib\": \"$lib\", \"rec\": /; s/\$/}/" >> $O
done; done
tail -2 gpurun_out/hint_pytest.log
