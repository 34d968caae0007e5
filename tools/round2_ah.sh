export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_srrsc.py -q -x -p no:cacheprovider > gpurun_out/round2_ah_t1.log 2>&1; echo "srrsc tests rc=$?"; grep -E "passed|failed|FAILED|Error|assert" gpurun_out/round2_ah_t1.log | head -10
timeout 600 python tools/adc1_bench.py 2>&1 | tail -3 | cut -c1-140
timeout 300 python tools/srrsc_prof.py 5000 64 3 2>&1 | tail -2
timeout 900 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/round2_ah_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/round2_ah_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('adc1', json.dumps(d.get('config4_adc1')))
for k,v in d.get('eigh',{}).items(): print(k, v.get('wall_s'))"
