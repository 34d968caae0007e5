export PYTHONUNBUFFERED=1
timeout 300 python tools/sanitize_small.py > gpurun_out/r04_san_plain.log 2>&1; echo "plain rc=$?"; tail -3 gpurun_out/r04_san_plain.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_small.py > gpurun_out/r04_san_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|sanitize driver done|Invalid|=========" gpurun_out/r04_san_memcheck.log | head -20
timeout 1200 $CS --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize_small.py merge > gpurun_out/r04_san_racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|sanitize driver done|hazard" gpurun_out/r04_san_racecheck.log | head -20
timeout 1200 $CS --tool synccheck --print-limit 50 python tools/sanitize_small.py merge > gpurun_out/r04_san_synccheck.log 2>&1; echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|sanitize driver done" gpurun_out/r04_san_synccheck.log | head -5
timeout 1200 $CS --tool initcheck --print-limit 30 python tools/sanitize_small.py merge > gpurun_out/r04_san_initcheck.log 2>&1; echo "initcheck rc=$?"; grep -E "ERROR SUMMARY|sanitize driver done|Uninitialized" gpurun_out/r04_san_initcheck.log | head -10
timeout 1500 $CS --tool memcheck --leak-check no --target-processes all --print-limit 30 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/r04_san_multirank.log 2>&1; echo "multirank memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r04_san_multirank.log | head -10
