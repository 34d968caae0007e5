export PYTHONUNBUFFERED=1 HSSEIG_NOPROF=1
for mb in 4 5 6 8; do
cp build/variants/lib_mb$mb.so paper_1510_04591_b200/libhsseig_b200.so
echo "== minb $mb"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wave_gather_kernel --csv --log-file gpurun_out/bp.csv python tools/eigh_prof.py 5 65536 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/bp.csv'))); hdr=None; t=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); t.append(float(d['Metric Value'].replace(',',''))/1e6)
print('top', t[-1], 'sum', sum(t[-12:]))
PY
done
