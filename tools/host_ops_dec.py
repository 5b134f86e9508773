"""Per-operation host cost (us, median of 2000) of the Python steps in front
of the first decode launch: python tools/host_ops_dec.py"""
import ctypes
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2508_10305_b200 as gz  # noqa: E402
from paper_2508_10305_b200 import _lib, pipeline as pl  # noqa: E402

torch.cuda.set_device(0)
x = torch.rand(1 << 20, device="cuda")
cont = gz.compress_device(gz.Dataset.from_axes([x, x, x]), gz.CompressConfig(error_bound=1e-3))
h = pl._known_header(cont)
cur = torch.cuda.current_stream()
ev = torch.cuda.Event()
s = pl._side_stream(0)
ops = {
    "current_stream": lambda: torch.cuda.current_stream(),
    "Event()+record": lambda: torch.cuda.Event().record(cur),
    "_side_stream": lambda: pl._side_stream(0),
    "wait_event": lambda: s.wait_event(ev),
    "_known_header": lambda: pl._known_header(cont),
    "torch.empty": lambda: torch.empty(3 * (1 << 20), dtype=torch.float32, device=x.device),
    "_workspace": lambda: pl._workspace(1 << 20, 0),
    "_device": lambda: pl._device(),
    "ptr_array": lambda: _lib.ptr_array([1, 2, 3]),
    "byref(h)": lambda: ctypes.byref(h),
    "cuda_stream": lambda: s.cuda_stream,
    "with stream(s)": lambda: torch.cuda.stream(s).__enter__(),
    "slice x3": lambda: [x[a * 10: a * 10 + 5] for a in range(3)],
    "Dataset._trusted": lambda: gz.Dataset._trusted((x, x, x), gz.Precision.F32),
    "ctypes 0-arg call": lambda: _lib.lib.gpzb_kernel_launches(),
}
for name, f in ops.items():
    ts = []
    for _ in range(2000):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    print("%-20s %6.2f us" % (name, statistics.median(ts) * 1e6))
    torch.cuda.synchronize()
