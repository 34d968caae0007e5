"""Per-launch durations in launch order from an ncu --csv launch list: python tools/ncu_seq.py file.csv [filter]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
flt = sys.argv[2] if len(sys.argv) > 2 else ""
hdr = None
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum" or flt not in d["Kernel Name"]:
            continue
        v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "nsecond" else 1.0)
        print(f"{d['ID']:>5} {v:10.1f} us  grid {d.get('Grid Size', '')}  {d['Kernel Name'][:90]}")
