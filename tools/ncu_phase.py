"""Aggregate an ncu cuda,sass source dump into per-line (file:line) totals and
print every line of one file with instruction share, for phase accounting."""
import csv
import sys


def main(path, fname):
    rows = list(csv.reader(open(path)))
    cur = "?"
    hdr = None
    per = {}
    tot = 0.0
    for r in rows:
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
            stl = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        tot += ins
        if cur == fname:
            per[int(d["Line No"])] = (ins, stl, r[1][:100])
    for ln in sorted(per):
        ins, stl, src = per[ln]
        if ins > 0 or stl > 0:
            print(f"{ln:4d} {100 * ins / tot:5.1f}% {stl:7.0f}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
