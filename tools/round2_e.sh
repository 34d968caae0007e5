export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/round2_e_mr.log 2>&1; echo "multirank rc=$?"; tail -2 gpurun_out/round2_e_mr.log
HSSEIG_ID_SMEM=1 timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/round2_e_mr_smem.log 2>&1; echo "multirank smem rc=$?"; tail -2 gpurun_out/round2_e_mr_smem.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_multirank.py > gpurun_out/round2_e_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_e_tests.log | head -20
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"id_" --csv \
  --log-file gpurun_out/round2_e_id.csv python tools/prof_merge.py 32768 1 > /dev/null 2>&1; echo "ncu rc=$?"
HSSEIG_ID_SMEM=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"id_" --csv \
  --log-file gpurun_out/round2_e_id_smem.csv python tools/prof_merge.py 32768 1 > /dev/null 2>&1; echo "ncu rc=$?"
