export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python tools/flops_probe.py 2>&1 | head -2
