"""Per-launch durations from an ncu --csv log: python tools/lv.py file.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
tot = 0.0
for r in rows:
    if 'Metric Name' in r:
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d['Metric Name'] != 'gpu__time_duration.sum':
            continue
        v = float(d['Metric Value']) / 1e6
        tot += v
        print(d['ID'], d['Grid Size'], '%.3f ms' % v)
print('total %.2f ms' % tot)
