export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ap_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ap_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-eigh 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms'])"
