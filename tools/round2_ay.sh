export PYTHONUNBUFFERED=1
python tools/eigh_prof.py 2 10000 2>&1 | head -48
