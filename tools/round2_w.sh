export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_w_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_w_tests.log | head -20
timeout 600 python tools/prof_merge.py 32768 5 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:tma_gemm --launch-skip 33 --launch-count 17 --csv --log-file gpurun_out/round2_w_mult.csv \
  python tools/prof_merge.py 32768 2 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/round2_w_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/round2_w_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('value', d['value'], 'ms', d['ms_per_step'], 'gpu_launches', d['gpu_launches'])
for k,v in d.get('eigh',{}).items(): print(k, {x: v.get(x) for x in ('wall_s','wall_s_e2e')})"
