export PYTHONUNBUFFERED=1 HSSEIG_TRACE_SUMMARY=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
python tools/host_trace.py 5 65536
