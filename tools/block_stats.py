"""Geometry of the bench datasets' blocks at full size (experiments only):
per-axis log2 m and N, runs U and stream widths from sampled block headers."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_10305_b200 as gz  # noqa: E402

torch.cuda.set_device(0)
pos, vel = bench.gen_hacc(bench.PARTICLES, 280, torch.device("cuda"))
for name, ax in (("pos", pos), ("vel", vel)):
    c = gz.compress_device(gz.Dataset.from_axes(ax), gz.CompressConfig(error_bound=1e-3)).cpu().numpy()
    nb = int(c[38:46].view("<u8")[0])
    table = c[46:46 + 8 * (nb + 1)].view("<u8")
    base = 46 + 8 * (nb + 1)
    rows = []
    for i in np.random.default_rng(0).integers(0, nb, 2000):
        b = c[base + int(table[i]): base + int(table[i + 1])]
        U = int(b[4:8].view("<u4")[0])
        geo = [(int(b[8 + a * 13 + 8]), int(b[8 + a * 13 + 9: 8 + a * 13 + 13].view("<u4")[0])) for a in range(3)]
        w = list(b[47:50])
        rows.append((U, max(g[1] << g[0] for g in geo), sum(g[0] for g in geo), w[0], w[1], w[2]))
    r = np.array(rows)
    print(name, "U mean/max", r[:, 0].mean(), r[:, 0].max(), "| max N<<b: mean", r[:, 1].mean(), "max", r[:, 1].max(),
          "frac<=64", (r[:, 1] <= 64).mean(), "| sumb", np.bincount(r[:, 2]), "| wd", np.bincount(r[:, 3]),
          "wc", np.bincount(r[:, 4]), "wo", np.bincount(r[:, 5]))
