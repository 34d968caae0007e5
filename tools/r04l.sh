timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r04_all6.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r04_all6.log | head -20
timeout 600 python tools/c4_ranks.py 2>&1 | grep -E "level|multiply" | head -9
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-eigh > gpurun_out/r04_bench6.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r04_bench6.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms','flops']: print(k, json.dumps(d.get(k)))"
