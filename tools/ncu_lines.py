"""Stall samples per CUDA source line from an ncu report: python tools/ncu_lines.py rep.ncu-rep [kernel-substr] [N]."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.Counter()
text = {}
cur_file = None
func = ""
for line in out.splitlines():
    if line.startswith('"File Path"'):
        cur_file = line.split('","')[1].rstrip('"')
        continue
    if line.startswith('"Function Name"'):
        func = line.split('","')[1]
        continue
    if line.startswith('"Line No"'):
        continue
    if want and want not in func:
        continue
    try:
        r = next(csv.reader(io.StringIO(line)))
    except StopIteration:
        continue
    if len(r) < 5 or not r[0].isdigit():
        continue
    try:
        v = float(r[4] or 0)
    except ValueError:
        continue
    key = (cur_file.split("/")[-1], int(r[0]))
    agg[key] += v
    text[key] = r[1]
tot = sum(agg.values()) or 1
for (f, ln), v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}% {f}:{ln}  {text[(f, ln)].strip()[:90]}")
