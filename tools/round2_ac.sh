export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_ac_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_ac_tests.log | head
timeout 600 python tools/prof_merge.py 32768 5 2>&1 | tail -1
