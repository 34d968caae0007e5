timeout 600 python tools/c4_ranks.py > gpurun_out/r04_ranks.log 2>&1; echo "ranks rc=$?"; cat gpurun_out/r04_ranks.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tma_gemm --launch-skip 2 --launch-count 17 \
  -o gpurun_out/r04_mult_full python tools/c4_ranks.py > gpurun_out/r04_ncu_full.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r04_ncu_full.log
