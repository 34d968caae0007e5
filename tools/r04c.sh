timeout 1800 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_properties.py -q -p no:cacheprovider -s > gpurun_out/r04_acc.log 2>&1; echo "acc rc=$?"
grep -E "ACCEPTANCE|passed|failed|FAILED|Error" gpurun_out/r04_acc.log | tail -40
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r04_all2.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/r04_all2.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-eigh > gpurun_out/r04_bench2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r04_bench2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms','roofline']: print(k, json.dumps(d.get(k)))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:tma_gemm --csv \
  --log-file gpurun_out/r04_launches2.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-eigh \
  > gpurun_out/r04_ncu_launch2.log 2>&1; echo "ncu rc=$?"
