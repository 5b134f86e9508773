"""Host-side cost of the batched calls (cProfile over repeated calls on the
bench workload): python tools/host_prof.py"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_10305_b200 as gz  # noqa: E402

torch.cuda.set_device(0)


class A:
    workload = "hacc280m"
    particles = bench.WORKLOADS["hacc280m"]["particles"]


jobs, _ = bench.build_jobs(A, 1, 0, torch.device("cuda"), gz)
dss, cfg = [j.ds for j in jobs], jobs[0].cfg
conts = gz.compress_batch_device(dss, cfg)
for _ in range(3):
    gz.decompress_batch_device(conts)
torch.cuda.synchronize()
# host time to enqueue (no sync inside except the result reads)
for label, fn in (("compress", lambda: gz.compress_batch_device(dss, cfg)),
                  ("decompress", lambda: gz.decompress_batch_device(conts))):
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    for _ in range(20):
        fn()
    pr.disable()
    torch.cuda.synchronize()
    print(label, "wall per call", (time.perf_counter() - t0) / 20 * 1e3, "ms")
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
