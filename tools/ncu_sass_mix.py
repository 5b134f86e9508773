"""Opcode mix of an `ncu --page source --csv --print-source cuda,sass` dump,
overall and for chosen file:line ranges (e.g. gpzb_encode_narrow.cuh:341-420)."""
import collections
import csv
import sys


def main(path, *ranges):
    rows = list(csv.reader(open(path)))
    cur_file, cur_line, hdr = "?", 0, None
    tot = collections.Counter()
    per = collections.defaultdict(collections.Counter)
    sel = []
    for spec in ranges:
        f, lr = spec.split(":")
        a, b = (int(x) for x in lr.split("-"))
        sel.append((spec, f, a, b))
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[2] == "-":
            cur_line = int(r[0]) if r[0].isdigit() else 0
            continue
        op = r[3].split()[0] if r[3].split() else "?"
        if op.startswith("@"):
            op = r[3].split()[1]
        op = op.split(".")[0]
        try:
            n = float(r[7] or 0)
        except ValueError:
            continue
        tot[op] += n
        for spec, f, a, b in sel:
            if cur_file == f and a <= cur_line <= b:
                per[spec][op] += n
    T = sum(tot.values())
    print(f"total warp instructions {T:.3e}")
    print("  " + ", ".join(f"{o} {v / T * 100:.1f}%" for o, v in tot.most_common(25)))
    for spec, *_ in sel:
        c = per[spec]
        s = sum(c.values())
        print(f"{spec}: {s / T * 100:.1f}% -> " + ", ".join(f"{o} {v / T * 100:.2f}" for o, v in c.most_common(14)))


if __name__ == "__main__":
    main(*sys.argv[1:])
