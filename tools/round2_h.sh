# tests touching the sample draw, the N > 1 bench path on one GPU (gloo), and the multiply DRAM capture
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_h_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_h_tests.log | head -20
HSSEIG_BENCH_N=16384 HSSEIG_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/round2_h_bench2.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/round2_h_bench2.log | head -c 5000; echo
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:tma_gemm --launch-skip 33 --launch-count 17 --csv --log-file gpurun_out/round2_h_mult.csv \
  python tools/prof_merge.py 32768 2 > /dev/null 2>&1; echo "ncu rc=$?"
