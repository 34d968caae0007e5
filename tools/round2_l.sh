export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_l_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_l_tests.log | head -20
for r in 0 16 32 48; do HSSEIG_SPLIT_RESERVE=$r timeout 600 python tools/prof_merge.py 32768 4 2>&1 | tail -1; done
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-eigh > gpurun_out/round2_l_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/round2_l_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms','roofline']: print(k, json.dumps(d.get(k)))"
