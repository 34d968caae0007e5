export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_srrsc.py -q -p no:cacheprovider > gpurun_out/round2_ak_t1.log 2>&1; echo "srrsc tests rc=$?"; grep -E "passed|failed|FAILED|Error|assert" gpurun_out/round2_ak_t1.log | head -10
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_ak_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_ak_tests.log | head
