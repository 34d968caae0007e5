export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/round2_v_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/round2_v_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('value', d['value'], 'ms', d['ms_per_step'])
for k,v in d.get('eigh',{}).items(): print(k, {x: v.get(x) for x in ('wall_s','wall_s_e2e','orthogonality','ratio_to_reference')})"
