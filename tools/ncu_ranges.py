"""Bucket an ncu source-page dump (--page source --csv --print-source cuda,sass)
by line ranges of one file: tools/ncu_ranges.py src.csv file.cuh a-b:name ..."""
import csv
import sys

path, fname = sys.argv[1], sys.argv[2]
ranges = []
for spec in sys.argv[3:]:
    ab, name = spec.split(":")
    a, b = ab.split("-")
    ranges.append((int(a), int(b), name))
cur = "?"
hdr = None
tot_i = tot_s = 0.0
buck = {}
for r in csv.reader(open(path)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    d = dict(zip(hdr, r))
    if d.get("Address") != "-":
        continue
    try:
        ins = float(d.get("Instructions Executed", "0") or 0)
        st = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    tot_i += ins
    tot_s += st
    ln = int(d["Line No"])
    name = "other:" + cur
    if cur == fname:
        for a, b, nm in ranges:
            if a <= ln <= b:
                name = nm
                break
    i0, s0 = buck.get(name, (0.0, 0.0))
    buck[name] = (i0 + ins, s0 + st)
print(f"total {tot_i:.3e} warp instr, {tot_s:.0f} samples")
for k, (i, s) in sorted(buck.items(), key=lambda x: -x[1][0]):
    print(f"{k:28s} instr {100 * i / tot_i:5.1f}%  stalls {100 * s / tot_s:5.1f}%")
