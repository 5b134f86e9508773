"""Does a host memmove overlap a pinned H2D / D2H on this box?  Experiments only."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2508_10305_b200 import pipeline as P  # noqa: E402

n = 541 << 20
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
x = torch.empty(n, dtype=torch.uint8, pin_memory=True)
y = torch.empty(n, dtype=torch.uint8, pin_memory=True)
src = torch.empty(n, dtype=torch.uint8)
src.fill_(3)
x.fill_(1)
y.fill_(2)


def t_(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print("H2D alone %.2f" % t_(lambda: dev.copy_(x, non_blocking=True)))
print("D2H alone %.2f" % t_(lambda: x.copy_(dev, non_blocking=True)))
print("memmove alone %.2f" % t_(lambda: P._par_memmove(y.data_ptr(), src.data_ptr(), n)))
print("H2D + memmove %.2f" % t_(lambda: (dev.copy_(x, non_blocking=True), P._par_memmove(y.data_ptr(), src.data_ptr(), n))))
print("D2H + memmove %.2f" % t_(lambda: (x.copy_(dev, non_blocking=True), P._par_memmove(y.data_ptr(), src.data_ptr(), n))))


def chunked():
    C = P._CHUNK
    for o in range(0, n, C):
        m = min(C, n - o)
        P._par_memmove(y.data_ptr() + o, src.data_ptr() + o, m)
        dev[o:o + m].copy_(y[o:o + m], non_blocking=True)


print("chunked stage+H2D %.2f" % t_(chunked))


def chunked_t():
    C = P._CHUNK
    ts = []
    for o in range(0, n, C):
        m = min(C, n - o)
        t0 = time.perf_counter()
        P._par_memmove(y.data_ptr() + o, src.data_ptr() + o, m)
        t1 = time.perf_counter()
        dev[o:o + m].copy_(y[o:o + m], non_blocking=True)
        t2 = time.perf_counter()
        ts.append("%.2f/%.2f" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
    torch.cuda.synchronize()
    print(" ".join(ts))


chunked_t()

s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
dev2 = torch.empty(n, dtype=torch.uint8, device="cuda")


def bidir():
    with torch.cuda.stream(s1):
        dev.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        y.copy_(dev2, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


print("H2D || D2H (separate streams) %.2f" % t_(bidir))
