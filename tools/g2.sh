timeout 900 python -m pytest tests/test_gpu_reference_seam.py tests/test_gpu_parity.py -q -k "seam or tql2 or base_size or reference_build" > gpurun_out/r04_seam.log 2>&1; echo "seam rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/r04_seam.log | head -30
timeout 900 python tools/orth_bisect.py > gpurun_out/r04_orth.log 2>&1; echo "orth rc=$?"; cat gpurun_out/r04_orth.log
