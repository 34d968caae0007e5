nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r04_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r04_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r04_bench.log | head -c 3000
