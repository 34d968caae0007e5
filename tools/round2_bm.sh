export PYTHONUNBUFFERED=1 HSSEIG_TRACE_SUMMARY=1
for st in 4 8 16 32; do
echo "== HSS streams $st"
export HSSEIG_HSS_STREAMS=$st
for i in 1 2; do HSSEIG_METHOD=adc-srrsc python tools/host_trace.py 2 10000; done
for i in 1 2; do HSSEIG_METHOD=adc-rand python tools/host_trace.py 2 10000; done
done
