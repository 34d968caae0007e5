export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/bl.txt 2>&1; tail -2 gpurun_out/bl.txt
export HSSEIG_TRACE_SUMMARY=1
HSSEIG_METHOD=adc-srrsc python tools/host_trace.py 2 10000
HSSEIG_METHOD=adc-rand python tools/host_trace.py 2 10000
HSSEIG_METHOD=adc-rand python tools/host_trace.py 2 10000
python tools/host_trace.py 3 20000
