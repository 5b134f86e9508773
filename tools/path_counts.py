import sys, torch
sys.path.insert(0, ".")
import bench
import paper_2508_10305_b200 as gz
from paper_2508_10305_b200 import pipeline as P
torch.cuda.set_device(0)
pos, vel = bench.gen_hacc(bench.PARTICLES, 280, torch.device("cuda"))
for name, ax in (("pos", pos), ("vel", vel)):
    c = gz.compress_device(gz.Dataset.from_axes(ax), gz.CompressConfig(error_bound=1e-3))
    print(name, P.last_path_counts())
