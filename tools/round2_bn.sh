export PYTHONUNBUFFERED=1
timeout 300 python tools/srrsc_c4.py 32768 check 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:srrsc --launch-skip 8 --launch-count 8 --csv --log-file gpurun_out/bn_srrsc_lv.csv python tools/srrsc_c4.py 32768 > /dev/null 2>&1; echo rc=$?
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/bn_srrsc_lv.csv'))); hdr=None; out=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); out.append((d['Grid Size'],float(d['Metric Value'].replace(',',''))/1e3))
print("# round 2 (final): ADC1 (SRRSC) construction of a k = 32768 / leaf 128 system (tools/srrsc_c4.py), ncu durations per level launch (leaf level first), lazy rescaling + block-major search")
for g,t in out: print(f"{t:9.1f} us  grid {g}")
print(f"total {sum(t for _,t in out)/1e3:.1f} ms")
PY
