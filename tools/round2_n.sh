# tests, bench line, multiply DRAM capture for the current multiply source (launch-skip: second
# merge of prof_merge = 8 sample launches + 17 multiply launches of the first, then 8 sample)
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_n_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_n_tests.log | head -20
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:tma_gemm --launch-skip 33 --launch-count 17 --csv --log-file gpurun_out/round2_n_mult.csv \
  python tools/prof_merge.py 32768 2 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-eigh > gpurun_out/round2_n_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/round2_n_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms','roofline','e2e']: print(k, json.dumps(d.get(k)))"
