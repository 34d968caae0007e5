export PYTHONUNBUFFERED=1
timeout 900 python tools/eigh_bench.py 2 3 5 2>&1 | tail -5
