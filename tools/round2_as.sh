export PYTHONUNBUFFERED=1 HSSEIG_NOPROF=1
for sh in 24 14 18 34; do
echo "== shape $sh"
export HSSEIG_GATHER_SHAPE=$sh
python tools/eigh_prof.py 5 65536 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:wave_gather_kernel --csv --log-file gpurun_out/as_gather.csv python tools/eigh_prof.py 5 65536 > gpurun_out/as_ncu.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/as_gather.csv')))
hdr=None; t=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); t.append(float(d['Metric Value'].replace(',',''))/1e6)
print('top', t[-1], 'sum', sum(t[-12:]), [round(x,3) for x in t[-12:-4]])
PY
done
