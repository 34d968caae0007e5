export PYTHONUNBUFFERED=1
python tools/eigh_prof.py 5 8192 2>&1 | head -60
