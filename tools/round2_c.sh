# GPU suite + config-4 phase timing after a change
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/round2_c_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED|Error|assert" gpurun_out/round2_c_tests.log | head -20
timeout 600 python tools/c4_ranks.py 2>&1 | head -12
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-eigh > gpurun_out/round2_c_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/round2_c_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms']: print(k, json.dumps(d.get(k)))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"id_kernel|genB|inner_form|leaf_form" --csv \
  --log-file gpurun_out/round2_c_build.csv python tools/prof_merge.py 32768 1 > /dev/null 2>&1; echo "ncu rc=$?"
