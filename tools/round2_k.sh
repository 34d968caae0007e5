# GPU suite, smoke, the default bench line (both arms)
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_k_tests.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/round2_k_tests.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/round2_k_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/round2_k_bench.log > gpurun_out/round2_k_bench.json
tail -1 gpurun_out/round2_k_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms','roofline','e2e','same_n','cpu_baseline']: print(k, json.dumps(d.get(k)))
for k,v in d.get('eigh',{}).items(): print(k, {x: v.get(x) for x in ('wall_s','wall_s_e2e','orthogonality','ratio_to_reference')})"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/round2_k_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/round2_k_ref.log
