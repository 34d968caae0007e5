"""Summarise the hottest SASS instructions of an ncu report: python tools/ncu_hot.py rep.ncu-rep [N]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for blk in blocks[1:]:
    lines = blk.splitlines()
    name = lines[0][:90]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = []
    tot = 0
    for r in rows[1:]:
        if len(r) != len(h):
            continue
        try:
            v = float(r[iss] or 0)
        except ValueError:
            continue
        tot += v
        data.append((v, r[ia], r[isrc]))
    data.sort(reverse=True)
    print("==", name, "samples", tot)
    for v, a, s in data[:top]:
        print(f"{100 * v / max(tot, 1):6.2f}% {a} {s}")
