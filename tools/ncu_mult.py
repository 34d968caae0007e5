"""Per-launch time, DMMA pipe and DRAM bytes of the multiply launches: python tools/ncu_mult.py file.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, d, order = None, {}, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        key = (int(x["ID"]), x["Kernel Name"][:70])
        if key not in d:
            d[key] = {}
            order.append(key)
        d[key][x["Metric Name"]] = (float(x["Metric Value"]), x["Metric Unit"])
tot = 0.0
for key in order:
    m = d[key]
    t, u = m["gpu__time_duration.sum"]
    t = t / 1e6 if u == "nsecond" else (t / 1e3 if u == "usecond" else t)
    tot += t
    dm = m.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", (0, ""))[0]
    rd = m.get("dram__bytes_read.sum", (0, "byte"))
    wr = m.get("dram__bytes_write.sum", (0, "byte"))
    sc = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}
    print(f"{key[0]:4d} {t:7.3f} ms dmma {dm:5.1f}% R {rd[0] * sc.get(rd[1], 1):6.2f} GB "
          f"W {wr[0] * sc.get(wr[1], 1):6.2f} GB {key[1][20:70]}")
print(f"total {tot:.3f} ms")
