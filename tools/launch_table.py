"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per kernel
name, launch count and per-launch durations (us)."""
import collections
import csv
import sys

d = collections.defaultdict(list)
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        if x.get('Metric Name') == 'gpu__time_duration.sum':
            d[x['Kernel Name'].split('(')[0][:48]].append(float(x['Metric Value'].replace(',', '')))
unit = 1e3 if len(sys.argv) < 3 else float(sys.argv[2])
for k, v in d.items():
    if 'gpzb' in k:
        print(f"{k:48s} n={len(v):3d} " + " ".join(f"{t / unit:.3f}" for t in v[:8]))
