"""Per-launch time and DRAM bytes from an ncu --csv list: python tools/ncu_mem.py file.csv [filter]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
flt = sys.argv[2] if len(sys.argv) > 2 else "hsseig"
hdr, d, order = None, {}, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        key = (x["ID"], x["Kernel Name"][:80])
        if key not in d:
            d[key] = {}
            order.append(key)
        d[key][x["Metric Name"]] = (float(x["Metric Value"]), x["Metric Unit"])
for key in order:
    if flt not in key[1]:
        continue
    m = d[key]
    t = m.get("gpu__time_duration.sum", (0, ""))
    rd = m.get("dram__bytes_read.sum", (0, ""))
    wr = m.get("dram__bytes_write.sum", (0, ""))
    print(f"{key[0]:>5} {t[0]:10.1f} {t[1]:8s} R {rd[0]:8.2f} {rd[1]:6s} W {wr[0]:8.2f} {wr[1]:6s} {key[1]}")
