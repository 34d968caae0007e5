set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r03_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r03_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r03_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r03_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r03_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r03_ref.log
