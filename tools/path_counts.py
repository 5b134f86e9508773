"""Blocks per encoder path (include/gpzb.h gpzb_encode_path_counts) of each
dataset of a bench workload: python tools/path_counts.py [workload]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_10305_b200 as gz  # noqa: E402
from paper_2508_10305_b200 import pipeline as P  # noqa: E402

torch.cuda.set_device(0)
wl = sys.argv[1] if len(sys.argv) > 1 else "hacc280m"


class A:
    workload = wl
    particles = bench.WORKLOADS[wl]["particles"]


jobs, _ = bench.build_jobs(A, 1, 0, torch.device("cuda"), gz)
print("paths: 0 no-offset K2/K2p, 1 composite, 2 in-group, 3 LSD, 4 general, 5 group masks, 6 K2s, 7 K2s offset-free")
for j in jobs:
    gz.compress_device(j.ds, j.cfg)
    print(wl, j.name, P.last_path_counts())
