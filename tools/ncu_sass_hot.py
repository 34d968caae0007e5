"""Top SASS instructions by warp-stall samples with their dominant reasons, from an
ncu --page source --csv --print-source sass export: python tools/ncu_sass_hot.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
i_ex = hdr.index("Instructions Executed")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[i_s] or 0) for r in data)
agg = {}
for i in st:
    agg[hdr[i]] = sum(int(r[i] or 0) for r in data)
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
order = sorted(range(len(data)), key=lambda j: -int(data[j][i_s] or 0))
for j in order[:top]:
    r = data[j]
    rs = sorted(((int(r[i] or 0), hdr[i][6:]) for i in st), reverse=True)[:3]
    print(f"{j:5d} {100 * int(r[i_s]) / tot:5.1f}%  ex {r[i_ex]:>9}  {r[i_src].strip()[:60]:60s} " +
          " ".join(f"{n}:{v}" for v, n in rs if v))
