"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel:
python tools/ncu_table.py file.csv [substring filter, e.g. hsseig]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        if len(sys.argv) > 2 and sys.argv[2] not in d["Kernel Name"]:
            continue
        name = d["Kernel Name"].split("(")[0][:60]
        v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "nsecond" else 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1] / 1e6:9.3f} ms {100 * v[1] / tot:5.1f}% {v[0]:5d}  {k}")
print(f"total {tot / 1e6:.3f} ms")
