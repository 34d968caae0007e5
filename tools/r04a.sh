# Round-2 re-entry: tests, smoke, bench (both arms), launch list on one B200.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/r04_all.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r04_all.log | tail -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r04_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r04_smoke.log
timeout 1500 python bench.py > gpurun_out/r04_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r04_bench.log > gpurun_out/r04_bench.json
tail -1 gpurun_out/r04_bench.log | head -c 6000; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r04_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r04_ref.log
