# One GPU session of the round's evidence: tests, smoke, bench (both arms), launch list.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r03_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r03_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r03_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r03_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r03_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r03_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:hsseig --csv \
  --log-file gpurun_out/r03_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-eigh \
  > gpurun_out/r03_ncu_launch.log 2>&1; echo "ncu rc=$?"
