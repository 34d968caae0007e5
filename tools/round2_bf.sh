export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/bf.txt 2>&1; tail -2 gpurun_out/bf.txt
python tools/flops_probe.py 2>&1 | head -2
