"""Per-source-line warp-instruction and stall shares from an
`ncu --page source --csv --print-source cuda,sass` dump (one kernel).

    python tools/ncu_lines.py src.csv [file-substring] [min-share-%]
"""
import csv
import sys


def main(path, want="", min_share=0.3):
    rows = list(csv.reader(open(path)))
    cur, fn, hdr = "?", "?", None
    per = {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) == 2 and r[0] == "Function Name":
            fn = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[2] != "-":
            continue
        try:
            ins = float(r[hdr.index("Instructions Executed")] or 0)
            st = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        k = (fn, cur, int(r[0]) if r[0].isdigit() else 0)
        a = per.setdefault(k, [0.0, 0.0, r[1]])
        a[0] += ins
        a[1] += st
    fns = sorted({k[0] for k in per})
    for f in fns:
        items = {k: v for k, v in per.items() if k[0] == f}
        ti = sum(v[0] for v in items.values()) or 1
        ts = sum(v[1] for v in items.values()) or 1
        print(f"== {f}: {ti:.4g} warp instructions, {ts:.4g} stall samples")
        byfile = {}
        for k, v in items.items():
            b = byfile.setdefault(k[1], [0, 0])
            b[0] += v[0]
            b[1] += v[1]
        for fl, v in sorted(byfile.items(), key=lambda x: -x[1][0]):
            print(f"   {fl:40s} instr {100 * v[0] / ti:5.1f}%  stalls {100 * v[1] / ts:5.1f}%")
        for k in sorted(items):
            v = items[k]
            if want and want not in k[1]:
                continue
            if 100 * v[0] / ti < min_share and 100 * v[1] / ts < min_share:
                continue
            print(f"{k[1][:22]:22s}:{k[2]:<5d} {100 * v[0] / ti:5.1f}% {100 * v[1] / ts:5.1f}%  {v[2].strip()[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", float(sys.argv[3]) if len(sys.argv) > 3 else 0.3)
