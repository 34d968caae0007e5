timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r04_all3.log 2>&1; echo "all rc=$?"; tail -2 gpurun_out/r04_all3.log
timeout 600 python tools/c4_ranks.py > gpurun_out/r04_ranks2.log 2>&1; grep multiply gpurun_out/r04_ranks2.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-eigh > gpurun_out/r04_bench3.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r04_bench3.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms','roofline']: print(k, json.dumps(d.get(k)))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:tma_gemm --csv \
  --log-file gpurun_out/r04_launches3.csv python tools/c4_ranks.py > /dev/null 2>&1; echo "ncu rc=$?"
