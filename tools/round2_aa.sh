export PYTHONUNBUFFERED=1
HSSEIG_NVCC_EXTRA=-DHSSEIG_ID_TIMING timeout 600 python -c "from paper_1510_04591_b200 import build as b; b.build(force=True)" 2>&1 | tail -2
timeout 300 python tools/id_timing.py 2>&1 | tail -8
