export PYTHONUNBUFFERED=1 HSSEIG_TRACE_SUMMARY=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "solver or baseline or fullsize or multirank or adc or seam or acceptance" > gpurun_out/bb.txt 2>&1; tail -2 gpurun_out/bb.txt
python tools/host_trace.py 5 65536 >> gpurun_out/bb.txt; python tools/host_trace.py 5 65536 >> gpurun_out/bb.txt; tail -2 gpurun_out/bb.txt
