export PYTHONFAULTHANDLER=1
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/r04_mr.log 2>&1; echo "mr rc=$?"; grep -E "passed|failed|Fatal|File|line" gpurun_out/r04_mr.log | head -40
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/r04_all3.log 2>&1; echo "all3 rc=$?"; grep -E "passed|failed|FAILED|cfg|c4_|max\||flops|ranks" gpurun_out/r04_all3.log | head -80
