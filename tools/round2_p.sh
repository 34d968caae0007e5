export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"id_kernel" --launch-skip 7 --launch-count 1 \
  -o gpurun_out/round2_id_top python tools/prof_merge.py 32768 1 > gpurun_out/round2_p_ncu.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/
