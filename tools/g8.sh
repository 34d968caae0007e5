timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r04_all4.log 2>&1; echo "all4 rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r04_all4.log | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r04_bench3.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r04_bench3.log > gpurun_out/r04_bench3.json; python -c "
import json; d=json.load(open('gpurun_out/r04_bench3.json'))
for k in ['value','ms_per_step','value_own_tree','phases_ms','flops','flops_reference','roofline','e2e','same_n','cpu_baseline','hss_rank']: print(k, json.dumps(d.get(k)))
for k,v in d.get('eigh',{}).items(): print(k, json.dumps(v))
"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r04_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r04_ref.log
