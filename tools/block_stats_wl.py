"""Block geometry of a bench workload's datasets from sampled block headers
of the GPU container: U (runs), Π N, Σ log2 m and the stream widths.
    python tools/block_stats_wl.py [workload]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_10305_b200 as gz  # noqa: E402

torch.cuda.set_device(0)
wl = sys.argv[1] if len(sys.argv) > 1 else "hacc280m"


class A:
    workload = wl
    particles = bench.WORKLOADS[wl]["particles"]


jobs, _ = bench.build_jobs(A, 1, 0, torch.device("cuda"), gz)
for j in jobs:
    c = gz.compress_device(j.ds, j.cfg).cpu().numpy()
    dims = j.ds.dims
    nb = int(c[38:46].view("<u8")[0])
    table = c[46:46 + 8 * (nb + 1)].view("<u8")
    base = 46 + 8 * (nb + 1)
    rows = []
    for i in np.random.default_rng(0).integers(0, nb, 4000):
        b = c[base + int(table[i]): base + int(table[i + 1])]
        U = int(b[4:8].view("<u4")[0])
        geo = [(int(b[8 + a * 13 + 8]), int(b[8 + a * 13 + 9: 8 + a * 13 + 13].view("<u4")[0])) for a in range(dims)]
        h = 8 + dims * 13
        w = list(b[h:h + 3])
        pn = int(np.prod([g[1] for g in geo]))
        rows.append((U, pn, sum(g[0] for g in geo), w[0], w[1], w[2]))
    r = np.array(rows)
    print(wl, j.name, "U mean", r[:, 0].mean().round(1), "| PN mean", r[:, 1].mean().round(0), "max", r[:, 1].max(),
          "| sumb", np.bincount(r[:, 2]).tolist(), "| wd", np.bincount(r[:, 3]).tolist(),
          "wc", np.bincount(r[:, 4]).tolist(), "wo", np.bincount(r[:, 5]).tolist())
    print("  K2s limits: sumb > 4 in %.2f%%, PN > 32768 in %.2f%%, both %.2f%%; PN histogram (2^k)" % (
        100 * (r[:, 2] > 4).mean(), 100 * (r[:, 1] > 32768).mean(), 100 * ((r[:, 2] > 4) & (r[:, 1] > 32768)).mean()),
        np.bincount(np.ceil(np.log2(np.maximum(r[:, 1], 1))).astype(int)).tolist())
    print("  paths", gz.pipeline.last_path_counts())
