export PYTHONUNBUFFERED=1 HSSEIG_NOPROF=1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "solver or multirank or baseline or adc or fullsize" > gpurun_out/ar_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ar_tests.log
for i in 1 2 3; do python tools/eigh_prof.py 5 65536 2>&1 | tail -1; done
python tools/eigh_prof.py 1 2000 2>&1 | tail -1
python tools/eigh_prof.py 3 20000 2>&1 | tail -1
python tools/eigh_prof.py 2 10000 2>&1 | tail -1
python tools/wave_prof.py 5 65536 2>&1 | head -30
