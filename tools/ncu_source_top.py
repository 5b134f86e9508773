"""Summarise an `ncu --page source --csv --print-source cuda,sass` dump:
top CUDA source lines by executed warp instructions and by stall samples."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur_file = "?"
    hdr = None
    agg = []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
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
        agg.append((cur_file, d["Line No"], ins, st, r[1][:90]))
    tot_i = sum(a[2] for a in agg) or 1
    tot_s = sum(a[3] for a in agg) or 1
    print(f"total warp instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
    print("--- by instructions")
    for f, ln, ins, st, src in sorted(agg, key=lambda a: -a[2])[:top]:
        print(f"{100*ins/tot_i:5.1f}% {100*st/tot_s:5.1f}%  {f}:{ln:5s} {src}")
    print("--- by stall samples")
    for f, ln, ins, st, src in sorted(agg, key=lambda a: -a[3])[:top]:
        print(f"{100*ins/tot_i:5.1f}% {100*st/tot_s:5.1f}%  {f}:{ln:5s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
