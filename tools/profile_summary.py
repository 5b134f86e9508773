"""Summarise ncu artefacts from gpurun_out/ into profiles/ (tracked).

usage: python tools/profile_summary.py <round-tag> [name=report.ncu-rep ...] [--launches launches.csv]

Writes profiles/<tag>_ncu_summary.json (+ .md): per captured kernel the
duration, DRAM bytes, instructions, issue/occupancy and top stall reasons;
and, from the `--metrics gpu__time_duration.sum` launch list, every kernel's
launch count, total and share of GPU time.  profiles/ncu_summary.json (the
file bench.py reads for `roofline.traffic`) is refreshed from the K2 capture.
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _num(v):
    return float(str(v).replace(",", ""))


def raw(path):
    """First profiled launch (dict) + units; numeric metrics averaged over all launches in the report."""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    h = next(r)
    units = next(r)
    rows = [dict(zip(h, v)) for v in r if v]
    d = dict(rows[0])
    for k in h:
        try:
            vals = [_num(x[k]) for x in rows]
        except (ValueError, KeyError):
            continue
        d[k] = str(sum(vals) / len(vals))
    d["_launches"] = len(rows)
    return d, dict(zip(h, units))


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return _num(v) * scale


def to_ms(v, unit):
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    return _num(v) * scale


def kernel_summary(path):
    d, u = raw(path)
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): _num(d[k]) for k in d
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and d[k]}
    tot = sum(st.values()) or 1
    rd = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
    wr = to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
    return {
        "kernel": d.get("Kernel Name") or d.get("Function Name", "?"),
        "duration_ms": to_ms(d["gpu__time_duration.sum"], u["gpu__time_duration.sum"]),
        "dram_read_bytes": rd,
        "dram_write_bytes": wr,
        "dram_bytes_per_launch": rd + wr,
        "dram_throughput_pct_of_peak": _num(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "0") or 0),
        "warp_instructions": _num(d["smsp__inst_executed.sum"]),
        "issue_active_pct": _num(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
        "warps_active_pct": _num(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
        "registers_per_thread": d.get("launch__registers_per_thread"),
        "grid": d.get("launch__grid_size"),
        "launches_averaged": d.get("_launches"),
        "top_stalls_pct": {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]},
    }


def launch_list(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = csv.DictReader(io.StringIO("".join(lines)))
    agg = {}
    for row in r:
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = row["Kernel Name"].split("(")[0]
        if "gpzb" not in name and "k_" not in name:
            name = "torch/other: " + name[:60]
        ns = to_ms(row["Metric Value"], row["Metric Unit"]) * 1e6
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    total = sum(v[1] for v in agg.values()) or 1
    for name, (cnt, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
        rows.append({"kernel": name, "launches": cnt, "total_ms": ns / 1e6, "avg_ms": ns / cnt / 1e6,
                     "share_pct": round(100 * ns / total, 2)})
    return rows


def main():
    tag = sys.argv[1]
    out = {"captures": {}, "launches": None}
    args = sys.argv[2:]
    i = 0
    while i < len(args):
        a = args[i]
        if a == "--launches":
            out["launches"] = launch_list(args[i + 1])
            i += 2
            continue
        name, path = a.split("=", 1)
        out["captures"][name] = kernel_summary(path)
        i += 1
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.json"), "w") as f:
        json.dump(out, f, indent=1)
    md = [f"# ncu summary {tag}", ""]
    for name, s in out["captures"].items():
        md.append(f"## {name}: {s['kernel'][:80]}")
        md.append(f"- duration {s['duration_ms']:.3f} ms (ncu, cold cache, clocks as running); DRAM read "
                  f"{s['dram_read_bytes'] / 1e9:.3f} GB, write {s['dram_write_bytes'] / 1e9:.3f} GB; "
                  f"DRAM throughput {s['dram_throughput_pct_of_peak']:.1f}% of peak")
        md.append(f"- warp instructions {s['warp_instructions']:.3e}; issue active {s['issue_active_pct']:.1f}%; "
                  f"warps active {s['warps_active_pct']:.1f}%; registers {s['registers_per_thread']}; grid {s['grid']}")
        md.append(f"- stalls: {s['top_stalls_pct']}")
        md.append("")
    if out["launches"]:
        md.append("## launch list (gpu__time_duration.sum, --clock-control none)")
        md.append("| kernel | launches | total ms | avg ms | share % |")
        md.append("|---|---|---|---|---|")
        for r in out["launches"][:20]:
            md.append(f"| {r['kernel'][:70]} | {r['launches']} | {r['total_ms']:.3f} | {r['avg_ms']:.4f} | "
                      f"{r['share_pct']} |")
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    enc = out["captures"].get("encode")
    if enc:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
            json.dump({"round": tag, "encode": {"dram_bytes_per_launch": enc["dram_bytes_per_launch"],
                                                "capture": f"profiles/{tag}_ncu_summary.json"}}, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
