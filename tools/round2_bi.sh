export PYTHONUNBUFFERED=1 HSSEIG_TRACE_SUMMARY=1 HSSEIG_METHOD=adc-srrsc
for c in 1 512 1024 2048 4096; do
echo "== cols per CTA $c"
export HSSEIG_SRRSC_COLS_PER_CTA=$c
python tools/host_trace.py 2 10000
python tools/srrsc_c4.py 2>&1 | tail -2
done
