export PYTHONUNBUFFERED=1 HSSEIG_NOPROF=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled --csv --log-file gpurun_out/bk_cfg2.csv python tools/eigh_prof.py 2 10000 > /dev/null 2>&1; echo rc=$?
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/bk_cfg2.csv'))); hdr=None; out=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); out.append((d['Kernel Name'].split('(')[0].replace('void ','').replace('hsseig::','')[:44],d['Grid Size'],float(d['Metric Value'].replace(',',''))/1e3))
half=out[len(out)//2:]
print(len(half),'launches, total ms',sum(t for *_,t in half)/1e3)
by=collections.defaultdict(list)
for n,g,t in half: by[n].append((g,t))
for n,v in sorted(by.items(), key=lambda kv:-sum(t for _,t in kv[1]))[:16]:
    gs=collections.Counter(g for g,_ in v).most_common(3)
    print(f"{sum(t for _,t in v)/1e3:8.2f} ms {len(v):5d}  {n:44s} grids {gs}")
PY
