timeout 1200 python tools/orth_bisect.py c4 8192 > gpurun_out/r04_bis_c4b.log 2>&1; echo "c4 rc=$?"; cat gpurun_out/r04_bis_c4b.log | tail -9
timeout 1200 python -m pytest tests/test_gpu_baseline_configs.py -q -s > gpurun_out/r04_cfgs2.log 2>&1; echo "cfgs rc=$?"; grep -E "passed|failed|Error|assert|cfg|c4_|max\||flops" gpurun_out/r04_cfgs2.log | head -40
timeout 600 python -m pytest tests/test_gpu_reference_seam.py -q > gpurun_out/r04_seam2.log 2>&1; echo "seam rc=$?"; grep -E "passed|failed|Error|assert|diff" gpurun_out/r04_seam2.log | head -30
timeout 900 python bench.py --steps 5 --warmup 3 --no-eigh --no-cpu > gpurun_out/r04_bench2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r04_bench2.log | head -c 1500
