"""Per-CUDA-line warp stall samples by reason (barrier excluded unless asked) from an ncu report:
python tools/ncu_stalls.py rep.ncu-rep [N] [--with-barrier]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 25
with_bar = "--with-barrier" in sys.argv
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.Counter()
why = collections.defaultdict(collections.Counter)
text = {}
hdr = None
cur = None
for line in out.splitlines():
    if line.startswith('"File Path"'):
        cur = line.split('","')[1].rstrip('"').split("/")[-1]
        continue
    r = next(csv.reader(io.StringIO(line)), None)
    if not r:
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) != len(hdr):
        continue
    for k, v in zip(hdr, r):
        if k.startswith("stall_") and "Not Issued" not in k:
            if k == "stall_barrier" and not with_bar:
                continue
            try:
                x = float(v or 0)
            except ValueError:
                continue
            agg[(cur, int(r[0]))] += x
            why[(cur, int(r[0]))][k[6:]] += x
    text[(cur, int(r[0]))] = r[1]
tot = sum(agg.values()) or 1
for key, v in agg.most_common(top):
    rs = ", ".join(f"{k} {100 * x / tot:.1f}" for k, x in why[key].most_common(3) if x)
    print(f"{100 * v / tot:5.1f}% {key[0]}:{key[1]}  [{rs}]  {text[key].strip()[:70]}")
