"""Headline numbers of an ncu --set full raw dump (one kernel): duration,
instructions, issue activity, occupancy, DRAM bytes, stall mix."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    g = lambda k: float(d[k].replace(",", "")) if d.get(k) not in (None, "", "n/a") else float("nan")  # noqa: E731
    print(d.get("Kernel Name", "?")[:60])
    print(f"  duration {g('gpu__time_duration.sum') / 1e3:.1f} us, warp instr {g('smsp__inst_executed.sum'):.3e}, "
          f"issue active {g('sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f}%, "
          f"warps active {g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%, "
          f"regs {g('launch__registers_per_thread'):.0f}")
    print(f"  dram read {g('dram__bytes_read.sum') / 1e9:.3f} GB, write {g('dram__bytes_write.sum') / 1e9:.3f} GB, "
          f"dram {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f}% of peak")
    st = {k: g(k) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in st.values() if v == v)
    top = sorted(st.items(), key=lambda kv: -(kv[1] if kv[1] == kv[1] else 0))[:9]
    print("  stalls: " + ", ".join(f"{k[33:]} {v / tot * 100:.1f}%" for k, v in top))
