export PYTHONUNBUFFERED=1 HSSEIG_TRACE_SUMMARY=1
for ns in 4 6 8; do
echo "== streams $ns"
HSSEIG_DENSE_STREAMS=$ns python tools/host_trace.py 5 65536
HSSEIG_DENSE_STREAMS=$ns python tools/host_trace.py 5 65536
done
