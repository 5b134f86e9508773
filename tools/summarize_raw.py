"""profiles/<tag>_ncu_summary.{json,md} from the raw-page CSVs of
tools/gpu_round2.sh (one --set full capture per kernel) and its launch list.

    python tools/summarize_raw.py <tag> name=gpurun_out/<tag>_<name>_raw.csv ... [--launches L.csv]
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_gb": ("dram__bytes_read.sum", 1e-9),
    "dram_write_gb": ("dram__bytes_write.sum", 1e-9),
    "dram_pct_of_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "warp_instructions": ("smsp__inst_executed.sum", 1),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "smem_static_bytes": ("launch__shared_mem_per_block_static", 1),
}


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    out = {"kernel": d.get("Kernel Name", "?")}
    for k, (m, scale) in KEYS.items():
        v = num(d.get(m))
        if v is None:
            continue
        unit = u.get(m, "")
        if m == "gpu__time_duration.sum":  # ns / us / ms as reported
            scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1, "ms": 1, "nsecond": 1e-6}.get(unit, 1e-6)
        if m == "launch__shared_mem_per_block_static":
            scale = {"byte": 1, "Kbyte": 1e3, "KB": 1e3}.get(unit, 1)
        if m.startswith("dram__bytes"):
            scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1, "KB": 1e-6, "MB": 1e-3, "GB": 1}.get(unit, 1e-9)
        out[k] = round(v * scale, 6)
    st = {k[33:]: num(v) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued") and num(v)}
    tot = sum(st.values())
    out["stalls_pct"] = {k: round(v / tot * 100, 1) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]}
    return out


def launches(path):
    per = collections.defaultdict(list)
    hdr = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            x = dict(zip(hdr, r))
            if x.get("Metric Name") == "gpu__time_duration.sum" and "gpzb" in x["Kernel Name"]:
                per[x["Kernel Name"].split("(")[0]].append(num(x["Metric Value"]) / 1e3)
    tot = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "total_us": round(sum(v), 1), "share_pct": round(100 * sum(v) / tot, 1)}
            for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))}


def main():
    tag = sys.argv[1]
    caps, lpath = {}, None
    args = sys.argv[2:]
    i = 0
    while i < len(args):
        if args[i] == "--launches":
            lpath = args[i + 1]
            i += 2
            continue
        name, p = args[i].split("=", 1)
        caps[name] = summarize(p)
        i += 1
    res = {"tag": tag, "captures": caps}
    if lpath:
        res["launch_list"] = launches(lpath)
    jp = os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.json")
    json.dump(res, open(jp, "w"), indent=1)
    lines = [f"# ncu summary {tag}", ""]
    for name, c in caps.items():
        lines.append(f"## {name}: {c['kernel']}")
        lines.append(f"- duration {c.get('duration_ms')} ms (ncu: cold cache, serialised); DRAM read "
                     f"{c.get('dram_read_gb')} GB, write {c.get('dram_write_gb')} GB ({c.get('dram_pct_of_peak')}% of peak)")
        lines.append(f"- warp instructions {c.get('warp_instructions'):.4g}; issue active {c.get('issue_active_pct')}%; "
                     f"warps active {c.get('warps_active_pct')}%; registers {c.get('registers')}; grid {c.get('grid')} x "
                     f"{c.get('block')}; static smem {c.get('smem_static_bytes')} B")
        lines.append(f"- stalls: {c['stalls_pct']}")
        lines.append("")
    if lpath:
        lines.append("## launch list (the repo's kernels in one bench run under ncu: warm-up + 2 steps, serialised)")
        lines.append("| kernel | launches | total us | share |")
        lines.append("|---|---|---|---|")
        for k, v in res["launch_list"].items():
            lines.append(f"| {k} | {v['launches']} | {v['total_us']} | {v['share_pct']}% |")
    open(jp.replace(".json", ".md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
