# full ncu capture of one whole config-4 multiply (17 launches, second merge of prof_merge)
export PYTHONUNBUFFERED=1
timeout 300 python tools/prof_merge.py 32768 2 || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tma_gemm --launch-skip 33 --launch-count 17 \
  -o gpurun_out/round2_mult_full python tools/prof_merge.py 32768 2 > gpurun_out/round2_ncu_mult_full.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/round2_mult_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active > gpurun_out/round2_mult_raw.csv; echo "export rc=$?"
