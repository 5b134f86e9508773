"""Group an A/B log (tools/gpu_ab_multi.sh output) by workload and library:
python tools/ab_summary.py gpurun_out/<tag>_ab.txt"""
import collections
import re
import sys

d = collections.defaultdict(list)
cur = None
for line in open(sys.argv[1]):
    if line.startswith("=="):
        _, wl, _, lib = line.split()
        cur = (wl, lib.split("/")[-1])
    elif cur:
        m = re.findall(r"(comp [\d.]+ decomp [\d.]+ ms [\d.]+)|(\w+: enc [\d.]+ dec [\d.]+)", line)
        d[cur].append(" | ".join(a or b for a, b in m))
for k, v in sorted(d.items()):
    for x in v:
        print("%-10s %-10s %s" % (k[0], k[1], x))
