timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_seam.py -q -p no:cacheprovider > gpurun_out/r04_p5.log 2>&1; echo "p5 rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r04_p5.log | head -30
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r04_bench3.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r04_bench3.log > gpurun_out/r04_bench3.json; python -c "
import json; d=json.load(open('gpurun_out/r04_bench3.json'))
for k in ['value','ms_per_step','value_own_tree','phases_ms','flops','flops_reference','roofline','e2e','same_n','cpu_baseline','hss_rank']: print(k, json.dumps(d.get(k)))
for k,v in d.get('eigh',{}).items(): print(k, json.dumps(v))
"
tail -5 gpurun_out/r04_bench3.log | grep -i error
