"""Timeline of one compress_batch_device call on the bench workload: every
C-ABI launch call is bracketed by CUDA events on its stream (the first marks
when the stream reaches the call, the second when its kernels are done), as
ms from the call's start.  python tools/batch_timeline.py [workload]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_10305_b200 as gz  # noqa: E402
from paper_2508_10305_b200 import _lib, pipeline  # noqa: E402

torch.cuda.set_device(0)
wl = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] != "rev" else "hacc280m"


class A:
    workload = wl
    particles = bench.WORKLOADS[wl]["particles"]


jobs, _ = bench.build_jobs(A, 1, 0, torch.device("cuda"), gz)
dss, cfg = [j.ds for j in jobs], jobs[0].cfg
if "rev" in sys.argv:
    dss = dss[::-1]
marks = []
names = ["gpzb_decompress_async", "gpzb_decompress_result", "gpzb_workspace_reset_async", "gpzb_range_async", "gpzb_range_background_async", "gpzb_range_finish_async",
         "gpzb_encode_plan_async", "gpzb_encode_async", "gpzb_emit_async", "gpzb_compress_result"]
names = [n for n in names if hasattr(_lib.lib, n)]
orig = {n: getattr(_lib.lib, n) for n in names}


def wrap(n):
    f = orig[n]

    def g(*a):
        s = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        r = f(*a)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(s)
        marks.append((n, s.stream_id, e0, e1))
        return r
    return g


for _ in range(3):
    conts = pipeline.compress_batch_device(dss, cfg)
    pipeline.decompress_batch_device(conts)
torch.cuda.synchronize()
for n in names:
    setattr(_lib.lib, n, wrap(n))
    setattr(pipeline.lib, n, getattr(_lib.lib, n))
for label, fn in (("compress_batch_device", lambda: pipeline.compress_batch_device(dss, cfg)),
                  ("decompress_batch_device", lambda: pipeline.decompress_batch_device(conts))):
    marks.clear()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    out = fn()
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record()
    torch.cuda.synchronize()
    if label.startswith("compress"):
        conts = out
    print(f"{label}: total {t0.elapsed_time(t1):.3f} ms")
    for n, sid, e0, e1 in marks:
        print(f"  stream {sid % 1000:4d} {n:32s} {t0.elapsed_time(e0):7.3f} -> {t0.elapsed_time(e1):7.3f}")
