export PYTHONUNBUFFERED=1 HSSEIG_NOPROF=1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "solver or baseline or fullsize or multirank or adc or seam" 2>&1 | tail -1
python tools/host_trace.py 5 65536 > gpurun_out/at_c5.txt 2>&1; cat gpurun_out/at_c5.txt
for i in 1 2 3; do python tools/eigh_prof.py 2 10000 2>&1 | tail -1; done
python tools/host_trace.py 2 10000 > gpurun_out/at_c2.txt 2>&1; cat gpurun_out/at_c2.txt
