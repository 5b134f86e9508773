"""Host-side split of one decompress_batch_device (or, with the argument
"compress", compress_batch_device) call on the bench workload:
perf_counter stamps at the C-ABI calls (entry/exit), medians over 30 calls,
plus the device time of the whole call (CUDA events):
python tools/host_dec_split.py"""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_10305_b200 as gz  # noqa: E402
from paper_2508_10305_b200 import _lib, pipeline  # noqa: E402

torch.cuda.set_device(0)


class A:
    workload = "hacc280m"
    particles = bench.WORKLOADS["hacc280m"]["particles"]


jobs, _ = bench.build_jobs(A, 1, 0, torch.device("cuda"), gz)
dss, cfg = [j.ds for j in jobs], jobs[0].cfg
conts = gz.compress_batch_device(dss, cfg)
stamps = []
COMP = len(sys.argv) > 1 and sys.argv[1] == "compress"
names = (["gpzb_range_async", "gpzb_encode_plan_async", "gpzb_encode_async", "gpzb_compress_result", "gpzb_emit_async"]
         if COMP else ["gpzb_decompress_async", "gpzb_decompress_result"])
for name in names:
    f = getattr(_lib.lib, name)

    def wrap(*a, _f=f, _n=name):
        stamps.append((_n[5:] + ">", time.perf_counter()))
        r = _f(*a)
        stamps.append((_n[5:] + "<", time.perf_counter()))
        return r
    setattr(_lib.lib, name, wrap)
    setattr(pipeline.lib, name, wrap)
rows, dev = [], []
for _ in range(30):
    torch.cuda.synchronize()
    stamps.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    gz.compress_batch_device(dss, cfg) if COMP else gz.decompress_batch_device(conts)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    dev.append(e0.elapsed_time(e1))
    rows.append([(n, (s - t0) * 1e6) for n, s in stamps] + [("return", (t1 - t0) * 1e6)])
print("device ms (median):", statistics.median(dev))
for k in range(len(rows[0])):
    print("%-28s %8.1f us" % (rows[0][k][0], statistics.median(r[k][1] for r in rows)))
