"""SASS (with executed warp-instruction counts) attributed to source lines
[a, b] of one file in an ncu source dump (--print-source cuda,sass):
    tools/ncu_sass_range.py src.csv file.cuh a b"""
import csv
import sys

path, fname, a, b = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
cur_file, line, tot = None, None, 0.0
for r in csv.reader(open(path)):
    if len(r) == 2 and r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]
        continue
    if not r or r[0] == 'Line No' or len(r) < 8:
        continue
    if r[0]:
        line = int(r[0]) if r[0].isdigit() else None
        if cur_file == fname and line is not None and a <= line <= b:
            print(f"---- {line}: {r[1].strip()[:100]}")
        continue
    if cur_file == fname and line is not None and a <= line <= b:
        try:
            ins = float(r[7] or 0)
        except ValueError:
            ins = 0.0
        tot += ins
        print(f"   {ins:11.0f}  {r[3].strip()}")
print(f"total {tot:.4g}")
