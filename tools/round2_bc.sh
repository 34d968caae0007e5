export PYTHONUNBUFFERED=1
unset HSSEIG_NOPROF
HSSEIG_METHOD=adc-srrsc python tools/eigh_prof.py 2 10000 2>&1 | head -40 > gpurun_out/bc_prof.txt; cat gpurun_out/bc_prof.txt
