"""Experiment: look-back counters of a -DGPZB_DEBUG_STATS build on the bench data."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_10305_b200 as gz
from paper_2508_10305_b200._lib import lib

out = (ctypes.c_uint64 * 8)()
pos, vel = bench.gen_hacc(280_000_000, 280, torch.device("cuda", 0))
for name, axes in (("pos", pos), ("vel", vel)):
    ds = gz.Dataset.from_axes(axes)
    gz.compress_device(ds, gz.CompressConfig(1e-3))
    lib.gpzb_debug_counters(out, 1)
    gz.compress_device(ds, gz.CompressConfig(1e-3))
    torch.cuda.synchronize()
    lib.gpzb_debug_counters(out, 1)
    nb = (280_000_000 + 1023) // 1024
    print(name, "rounds/block %.3f spins/block %.3f dist %.2f" % (out[0] / nb, out[1] / nb, out[2] / nb), list(out))
