export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/round2_o_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED|Error|assert" gpurun_out/round2_o_tests.log | head -20
for r in 0 24 32 48; do echo "reserve $r"; HSSEIG_SPLIT_RESERVE=$r timeout 600 python tools/prof_merge.py 32768 5 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"id_kernel" --csv \
  --log-file gpurun_out/round2_o_id.csv python tools/prof_merge.py 32768 1 > /dev/null 2>&1; echo "ncu rc=$?"
