export PYTHONUNBUFFERED=1
timeout 600 python tools/e2e_probe.py 32768 16
timeout 600 python tools/e2e_probe.py 32768 32
