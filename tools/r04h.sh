timeout 300 python tools/sec_bench.py 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r04_all4.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED|assert" gpurun_out/r04_all4.log | head -20
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-eigh > gpurun_out/r04_bench4.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r04_bench4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms','roofline']: print(k, json.dumps(d.get(k)))"
