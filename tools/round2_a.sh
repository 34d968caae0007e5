# Round-2 (session 3) evidence: tests, smoke, bench (both arms), launch list on one B200.
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_gputests.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/round2_gputests.log | tail -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/round2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/round2_smoke.log
timeout 1500 python bench.py > gpurun_out/round2_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/round2_bench.log > gpurun_out/round2_bench.json
tail -1 gpurun_out/round2_bench.log | head -c 8000; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/round2_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/round2_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled --csv \
  --log-file gpurun_out/round2_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-eigh \
  > gpurun_out/round2_ncu_launch.log 2>&1; echo "ncu rc=$?"
