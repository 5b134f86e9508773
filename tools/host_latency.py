"""Host time from the call of compress_batch_device / decompress_batch_device
to its first C-ABI launch (the GPU idles meanwhile): python tools/host_latency.py"""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_10305_b200 as gz  # noqa: E402
from paper_2508_10305_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)


class A:
    workload = "hacc280m"
    particles = bench.WORKLOADS["hacc280m"]["particles"]


jobs, _ = bench.build_jobs(A, 1, 0, torch.device("cuda"), gz)
dss, cfg = [j.ds for j in jobs], jobs[0].cfg
conts = gz.compress_batch_device(dss, cfg)
stamps = []
for name in ("gpzb_decompress_async", "gpzb_workspace_reset_async"):
    f = getattr(_lib.lib, name)

    def wrap(*a, _f=f):
        stamps.append(time.perf_counter())
        return _f(*a)
    setattr(_lib.lib, name, wrap)
for label, fn in (("decompress", lambda: gz.decompress_batch_device(conts)),
                  ("compress", lambda: gz.compress_batch_device(dss, cfg))):
    lat = []
    for _ in range(30):
        torch.cuda.synchronize()
        stamps.clear()
        t0 = time.perf_counter()
        fn()
        lat.append([(s - t0) * 1e6 for s in stamps[:2]])
    print(label, "us to the 1st / 2nd launch call (median):",
          statistics.median(x[0] for x in lat), statistics.median(x[1] for x in lat))
