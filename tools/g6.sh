timeout 1800 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_baseline_configs.py -p no:cacheprovider > gpurun_out/r04_all.log 2>&1; echo "all rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/r04_all.log | head -30
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r04_all2.log 2>&1; echo "all2 rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r04_all2.log | head -60
timeout 1200 python tools/orth_bisect.py c4 8192 > gpurun_out/r04_bis_c4c.log 2>&1; tail -3 gpurun_out/r04_bis_c4c.log
