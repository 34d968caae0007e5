"""Turn an ncu csv of ONE config-4 multiply (17 tma_gemm launches of MergePipeline, captured
with gpu__time_duration / dram__bytes_read / dram__bytes_write) into
profiles/multiply_traffic.json, stamped with the multiply kernel source hash that bench.py
checks before it reports roofline.traffic:
  python tools/traffic_json.py gpurun_out/x.csv profiles/x.csv"""
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
src = b"".join(open(os.path.join(ROOT, "paper_1510_04591_b200", "csrc", f), "rb").read()
               for f in ("hss_mult.cu", "tma.cuh"))
sha = hashlib.sha256(src).hexdigest()[:16]
rows = list(csv.reader(open(sys.argv[1])))
sc = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
      "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
hdr, per = None, {}
if rows and "Metric Name" not in rows[0] and "gpu__time_duration.sum" in rows[0]:
    # `ncu -i rep --page raw --csv`: one row per launch, a units row under the header
    h, u = rows[0], rows[1]
    for n, r in enumerate(rows[2:]):
        per[n] = {k: float(r[h.index(k)].replace(",", "")) * sc.get(u[h.index(k)], 1.0)
                  for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum")}
for r in rows if not per else []:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        per.setdefault(int(x["ID"]), {})[x["Metric Name"]] = float(x["Metric Value"]) * sc.get(x["Metric Unit"], 1.0)
ids = sorted(per)
assert len(ids) == 17, f"expected the 17 launches of one multiply, got {len(ids)}"
rd = sum(per[i]["dram__bytes_read.sum"] for i in ids)
wr = sum(per[i]["dram__bytes_write.sum"] for i in ids)
t = sum(per[i]["gpu__time_duration.sum"] for i in ids)
out = {"file": os.path.basename(sys.argv[2]) if len(sys.argv) > 2 else sys.argv[1],
       "source_sha16": sha, "launches": 17, "bytes_read": rd, "bytes_write": wr,
       "bytes_per_multiply": rd + wr, "ncu_time_s": t,
       "algorithmic_bytes": 2 * 32768 * 32768 * 8,
       "note": "one whole config-4 multiply (P = 32768 rows in one call, MergePipeline), ncu kernel replay "
               "(cold caches); algorithmic = Q_old read once + Q_new written once"}
if len(sys.argv) > 2:
    import shutil
    shutil.copy(sys.argv[1], sys.argv[2])
json.dump(out, open(os.path.join(ROOT, "profiles", "multiply_traffic.json"), "w"), indent=1)
print(json.dumps(out))
