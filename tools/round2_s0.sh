# Session re-entry check at head: GPU suite, smoke, default bench line
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/s0_tests.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/s0_tests.log | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/s0_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s0_bench.log > gpurun_out/s0_bench.json
tail -1 gpurun_out/s0_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms','e2e','clocks']: print(k, json.dumps(d.get(k)))
for k,v in d.get('eigh',{}).items(): print(k, {x: v.get(x) for x in ('wall_s','wall_s_e2e')})"
