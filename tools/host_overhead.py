"""Host-side cost of the batched device calls (experiments only): wall time
of compress_batch_device / decompress_batch_device vs the device time of
their kernels, and the host time of each phase of the decompress batch."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_10305_b200 as gz  # noqa: E402
from paper_2508_10305_b200 import pipeline as P  # noqa: E402

torch.cuda.set_device(0)
pos, vel = bench.gen_hacc(bench.PARTICLES, 280, torch.device("cuda"))
ds = [gz.Dataset.from_axes(pos), gz.Dataset.from_axes(vel)]
cfg = gz.CompressConfig(error_bound=1e-3)
for _ in range(3):
    conts = gz.compress_batch_device(ds, cfg)
    recs = gz.decompress_batch_device(conts)
torch.cuda.synchronize()
for it in range(3):
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    t0 = time.perf_counter()
    a.record()
    conts = gz.compress_batch_device(ds, cfg)
    b.record()
    t1 = time.perf_counter()
    recs = gz.decompress_batch_device(conts)
    c.record()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"compress: events {a.elapsed_time(b):.3f} ms, host {1e3 * (t1 - t0):.3f} ms | decompress: events "
          f"{b.elapsed_time(c):.3f} ms, host {1e3 * (t2 - t1):.3f} ms")
# phases of the decompress batch, host clock
torch.cuda.synchronize()
marks = []
t0 = time.perf_counter()
launched = []
for i, data in enumerate(conts):
    s = P._side_stream(i)
    with torch.cuda.stream(s):
        ta = time.perf_counter()
        t, h = P._to_device_bytes(data)
        tb = time.perf_counter()
        launched.append(P._decode_launch(t, h, slot=i))
        tc = time.perf_counter()
        marks.append(f"hdr {1e3 * (tb - ta):.3f} launch {1e3 * (tc - tb):.3f}")
for i, L in enumerate(launched):
    with torch.cuda.stream(P._side_stream(i)):
        ta = time.perf_counter()
        P._decode_result(L)
        marks.append(f"result {1e3 * (time.perf_counter() - ta):.3f}")
print(" | ".join(marks), f"| total {1e3 * (time.perf_counter() - t0):.3f} ms")
