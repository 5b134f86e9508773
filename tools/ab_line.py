"""One summary line per bench JSON line on stdin (used by tools/gpu_ab_wl.sh)."""
import json
import sys

for line in sys.stdin:
    try:
        d = json.loads(line)
    except ValueError:
        continue
    pj = " ".join("%s: enc %.3f dec %.3f rng %.3f" % (k, v["encode_ms"], v["decode_ms"], v["range_ms"])
                  for k, v in d["per_job"].items())
    clk = d["clocks"]["sm_mhz"] if d.get("clocks") else None
    print("comp %.1f decomp %.1f ms %.3f | %s | clk %s" % (d["value"], d["decompress"]["value"], d["ms_per_step"], pj, clk))
