export PYTHONUNBUFFERED=1 HSSEIG_NOPROF=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "solver or baseline or fullsize or multirank or adc or seam or acceptance or halves" 2>&1 | tail -3
python tools/host_trace.py 5 65536 > gpurun_out/au_c5.txt 2>&1; cat gpurun_out/au_c5.txt
python tools/host_trace.py 1 2000 > gpurun_out/au_c1.txt; head -1 gpurun_out/au_c1.txt
python tools/host_trace.py 3 20000 > gpurun_out/au_c3.txt; head -1 gpurun_out/au_c3.txt
