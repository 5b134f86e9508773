"""Per-source-line warp-instruction counts for ONE function of an
`ncu --page source --csv --print-source cuda,sass` dump (the OCC-th report of
that function, default 1), all files, normalised by a count (e.g. warp-blocks):
tools/ncu_func_lines.py src.csv '<function substring>' norm [top]"""
import csv
import os
import sys

path, fsub, norm = sys.argv[1], sys.argv[2], float(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 60
cur_file, cur_fn, hdr, seen_n, out = "?", None, None, {}, {}
OCC = int(os.environ.get("OCC", "1"))  # which report of the function
active = False
for r in csv.reader(open(path)):
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) == 2 and r[0] == "Function Name":
        key = (r[1], cur_file)
        seen_n[key] = seen_n.get(key, 0) + 1
        active = fsub in r[1] and seen_n[key] == OCC
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not active or hdr is None or len(r) < 8 or r[2] != "-" or not r[0].isdigit():
        continue
    n = float(r[hdr.index("Instructions Executed")] or 0)
    if n:
        out[(cur_file, int(r[0]))] = (n, r[1].strip()[:80])
tot = sum(v[0] for v in out.values())
print("total %.4g warp instr = %.1f per norm unit" % (tot, tot / norm))
for (f, ln), (n, src) in sorted(out.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%6.1f  %s:%d  %s" % (n / norm, f, ln, src))
