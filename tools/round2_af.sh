# round-2 key-metric captures at the head: the two sampling GEMMs (first Y and Z^T chunk of the
# second merge), the top-level ID, the multiply's leaf finish, the secular kernel
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none -k regex:tma_gemm --launch-skip 24 --launch-count 2 \
  -o /tmp/rf_sample python tools/prof_merge.py 32768 2 > /dev/null 2>&1; echo "ncu sample rc=$?"
ncu -i /tmp/rf_sample.ncu-rep --page raw --csv > gpurun_out/rf_sample_raw.csv
timeout 900 ncu --set full --clock-control none -k regex:tma_gemm --launch-skip 47 --launch-count 1 \
  -o /tmp/rf_leaf python tools/prof_merge.py 32768 2 > /dev/null 2>&1; echo "ncu leaf rc=$?"
ncu -i /tmp/rf_leaf.ncu-rep --page raw --csv > gpurun_out/rf_leaf_raw.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:id_kernel --launch-skip 7 --launch-count 1 \
  -o gpurun_out/rf_id_top python tools/prof_merge.py 32768 1 > /dev/null 2>&1; echo "ncu id rc=$?"
ls -la gpurun_out | tail -5
