export PYTHONUNBUFFERED=1 HSSEIG_NOPROF=1 HSSEIG_METHOD=adc-srrsc
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:srrsc --csv --log-file gpurun_out/bh_srrsc.csv python tools/eigh_prof.py 2 10000 > /dev/null 2>&1; echo rc=$?
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/bh_srrsc.csv'))); hdr=None; out=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); out.append((d['Grid Size'],float(d['Metric Value'].replace(',',''))/1e3))
half=out[len(out)//2:]
print(len(half),'launches, total ms',sum(t for _,t in half)/1e3)
import collections
by=collections.defaultdict(list)
for g,t in half: by[g].append(t)
for g,ts in sorted(by.items(), key=lambda kv:-sum(kv[1])): print(g, len(ts), 'sum %.1f us'%sum(ts), 'max %.1f'%max(ts), 'mean %.1f'%(sum(ts)/len(ts)))
PY
