# acceptance + property suites on the GPU path, then the bench launch list (ncu, durations only)
timeout 1800 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_properties.py -q -p no:cacheprovider -s > gpurun_out/r04_acc.log 2>&1; echo "acc rc=$?"
grep -E "ACCEPTANCE|passed|failed|FAILED|Error" gpurun_out/r04_acc.log | tail -40
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:hsseig --csv \
  --log-file gpurun_out/r04_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-eigh \
  > gpurun_out/r04_ncu_launch.log 2>&1; echo "ncu rc=$?"
