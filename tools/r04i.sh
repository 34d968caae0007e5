timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r04_all5.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED|assert" gpurun_out/r04_all5.log | head -20
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-eigh > gpurun_out/r04_bench5.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r04_bench5.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms']: print(k, json.dumps(d.get(k)))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"gen_panel|tma_gemm|splitk|transpose" --csv \
  --log-file gpurun_out/r04_launches5.csv python tools/prof_merge.py 32768 1 > /dev/null 2>&1; echo "ncu rc=$?"
