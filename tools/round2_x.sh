export PYTHONUNBUFFERED=1
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/round2_x_mr$i.log 2>&1; echo "multirank $i rc=$?"; grep -E "passed|failed|SIGSEGV|Error" gpurun_out/round2_x_mr$i.log | tail -2; done
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_multirank.py > gpurun_out/round2_x_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_x_tests.log | head
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/round2_x_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/round2_x_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('value', d['value'], 'ms', d['ms_per_step'])
for k,v in d.get('eigh',{}).items(): print(k, {x: v.get(x) for x in ('wall_s','wall_s_e2e','glue_hbm')})"
