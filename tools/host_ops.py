"""Host cost of the individual steps of decompress_batch_device (us each,
median of 200): python tools/host_ops.py"""
import ctypes
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2508_10305_b200 as gz  # noqa: E402
from paper_2508_10305_b200 import _lib, pipeline as P  # noqa: E402
from oracle import gpz_oracle as O  # noqa: E402

torch.cuda.set_device(0)
axes = [torch.from_numpy(a).cuda() for a in O.gen_clusters(1 << 20, dims=3, seed=1)]
c = gz.compress_device(gz.Dataset.from_axes(axes), gz.CompressConfig(1e-3))
h = P._known_header(c)
s = P._side_stream(0)
cur = torch.cuda.current_stream()
ev = torch.cuda.Event()
ws = P._workspace(1 << 26, 0)
outs = [torch.empty(1 << 20, device="cuda") for _ in range(3)]


def t(label, fn, n=200):
    xs = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        xs.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    print(f"{label:40s} {statistics.median(xs):8.2f} us")


def ctx():
    with torch.cuda.stream(s):
        pass


t("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
t("Event() + record", lambda: torch.cuda.Event().record(cur))
t("_side_stream(0)", lambda: P._side_stream(0))
t("s.wait_event(ev)", lambda: s.wait_event(ev))
t("with torch.cuda.stream(s)", ctx)
t("_to_device_bytes(c)", lambda: P._to_device_bytes(c))
t("torch.empty(3 * 2^20 f32)", lambda: torch.empty(3 << 20, device="cuda"))
t("_workspace(2^20)", lambda: P._workspace(1 << 20, 0))
t("_stream()", lambda: P._stream())
t("ptr_array(3)", lambda: _lib.ptr_array([1, 2, 3]))
t("Precision(0)", lambda: gz.Precision(0))
hp = ctypes.byref(h)
arr = _lib.ptr_array([o.data_ptr() for o in outs])
t("gpzb_decompress_async (C, 3 launches)", lambda: _lib.lib.gpzb_decompress_async(
    c.data_ptr(), c.numel(), hp, arr, 1 << 20, None, ws.data_ptr(), ws.numel(), s.cuda_stream), n=50)
t("_decode_launch (all)", lambda: P._decode_launch(c, h, slot=0, stream=s.cuda_stream), n=50)
t("decompress_batch_device([c]) incl. sync", lambda: gz.decompress_batch_device([c]), n=20)
