export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fused_leaf or multiply or matmul or hss" > gpurun_out/round2_ae_t1.log 2>&1; echo "t1 rc=$?"; grep -E "passed|failed|FAILED|Error|assert" gpurun_out/round2_ae_t1.log | head -10
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_ae_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_ae_tests.log | head
for f in 0 1; do HSSEIG_LEAF_FUSED=$f timeout 600 python tools/prof_merge.py 32768 5 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"tma_leaf|tma_gemm" --launch-skip 33 --launch-count 16 --csv --log-file gpurun_out/round2_ae_mult.csv \
  python tools/prof_merge.py 32768 2 > /dev/null 2>&1; echo "ncu rc=$?"
