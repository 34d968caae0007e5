# compute-sanitizer passes on small shapes (one tool at a time, after a clean plain run),
# the secular kernel's full ncu capture and the multiply's DRAM traffic (17 launches).
export PYTHONUNBUFFERED=1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_small.py > gpurun_out/round2_san_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/round2_san_plain.log
timeout 1500 $CS --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_small.py > gpurun_out/round2_san_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|sanitize driver done" gpurun_out/round2_san_memcheck.log | head
timeout 1200 $CS --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize_small.py merge > gpurun_out/round2_san_racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|sanitize driver done" gpurun_out/round2_san_racecheck.log | head
timeout 900 $CS --tool synccheck --print-limit 50 python tools/sanitize_small.py merge > gpurun_out/round2_san_synccheck.log 2>&1; echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|sanitize driver done" gpurun_out/round2_san_synccheck.log | head
timeout 900 $CS --tool initcheck --print-limit 30 python tools/sanitize_small.py merge > gpurun_out/round2_san_initcheck.log 2>&1; echo "initcheck rc=$?"; grep -E "ERROR SUMMARY|sanitize driver done" gpurun_out/round2_san_initcheck.log | head
timeout 900 $CS --tool memcheck --leak-check no --target-processes all --print-limit 30 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/round2_san_multirank.log 2>&1; echo "multirank memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/round2_san_multirank.log | head
timeout 600 ncu --set full --clock-control none --import-source on -k regex:secular_queue --launch-skip 2 --launch-count 1 \
  -o gpurun_out/round2_secular python tools/sec_bench.py > gpurun_out/round2_ncu_sec.log 2>&1; echo "ncu sec rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum \
  --clock-control none -k regex:tma_gemm --launch-skip 25 --launch-count 17 --csv --log-file gpurun_out/round2_mult_traffic.csv \
  python tools/c4_ranks.py > gpurun_out/round2_ncu_mult.log 2>&1; echo "ncu mult rc=$?"
