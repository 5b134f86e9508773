"""Per-source-line warp-instruction counts of one file in an ncu source dump,
normalised by a reference line's count (e.g. a line executed once per block
per warp) or, with a leading '=', by a number (e.g. =1037588 warp-blocks):
tools/ncu_linecount.py src.csv file.cuh ref_line|=count"""
import csv
import sys

path, fname, ref = sys.argv[1], sys.argv[2], sys.argv[3]
cur, hdr, lines = "?", None, {}
for r in csv.reader(open(path)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or cur != fname or len(r) < 8 or r[2] != "-":
        continue
    try:
        lines[int(r[0])] = (float(r[hdr.index("Instructions Executed")] or 0), r[1].strip()[:90])
    except ValueError:
        pass
base = float(ref[1:]) if ref.startswith("=") else lines[int(ref)][0]
tot = 0
for ln in sorted(lines):
    n, src = lines[ln]
    if n:
        tot += n / base
        print(f"{ln:5d} {n / base:8.1f}  {src}")
print(f"total per ref-line execution: {tot:.0f} warp instructions")
