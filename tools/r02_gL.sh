cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "async or copy" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_abi_cpu.py -x -q 2>&1 | tail -1
timeout 900 python bench.py --no-configs --no-next2 --no-cpu-baseline > gpurun_out/gL_bench.jsonl 2> gpurun_out/gL_bench.err; python -c "
import json; l=[x for x in open('gpurun_out/gL_bench.jsonl') if x.startswith('{')][-1]; d=json.loads(l); print(d['value'], json.dumps(d['e2e'])[:900])"
