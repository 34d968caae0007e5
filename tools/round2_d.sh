# full ncu capture of one whole config-4 multiply (17 launches, second merge of prof_merge);
# the report stays in /tmp (too large to bring back), its raw page and per-line source
# stalls of two launches come back as CSV
export PYTHONUNBUFFERED=1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tma_gemm --launch-skip 33 --launch-count 17 \
  -o /tmp/round2_mult_full python tools/prof_merge.py 32768 2 > gpurun_out/round2_ncu_mult_full.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/round2_mult_full.ncu-rep --page raw --csv > gpurun_out/round2_mult_raw.csv; echo "export rc=$?"
ncu -i /tmp/round2_mult_full.ncu-rep --page source --csv --launch-skip 0 --launch-count 1 > gpurun_out/round2_mult_src_leafup.csv 2>&1; echo "src rc=$?"
ncu -i /tmp/round2_mult_full.ncu-rep --page source --csv --launch-skip 15 --launch-count 1 > gpurun_out/round2_mult_src_down8.csv 2>&1
ls -la gpurun_out/
