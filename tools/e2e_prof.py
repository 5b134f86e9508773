import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, numpy as np, ctypes
import bench, paper_2508_10305_b200 as gz
n = 280_000_000
pos, vel = bench.gen_hacc(n, 280, torch.device("cuda", 0))
host = [a.cpu().pin_memory() for a in pos]
cfg = gz.CompressConfig(1e-3)
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = T(); dev = [h.to("cuda", non_blocking=True) for h in host]; t1 = T()
    out = gz.compress_device(gz.Dataset.from_axes(dev), cfg); t2 = T()
    pin = torch.empty(out.numel(), dtype=torch.uint8, pin_memory=True); t3 = T()
    pin.copy_(out); t4 = T()
    b = pin.numpy().tobytes(); t5 = T()
    # pageable direct
    b2 = out.cpu().numpy().tobytes(); t6 = T()
    print(f"H2D {t1-t0:.4f} ({12*n/(t1-t0)/3e9:.1f} GB/s) comp {t2-t1:.4f} pinalloc {t3-t2:.4f} D2H {t4-t3:.4f} tobytes {t5-t4:.4f} pageable-path {t6-t5:.4f}")
    t0 = T(); hb = np.frombuffer(b, np.uint8); dt = torch.from_numpy(hb).to("cuda"); t1 = T()
    pin2 = torch.empty(len(b), dtype=torch.uint8, pin_memory=True); pin2.numpy()[:] = hb; t2 = T()
    dt2 = pin2.to("cuda", non_blocking=True); t3 = T()
    rec = gz.decompress_device(dt2); t4 = T()
    o = [a.cpu() for a in rec.axes]; t5 = T()
    o2 = [torch.empty(a.numel(), dtype=a.dtype, pin_memory=True) for a in rec.axes]; t6 = T()
    for x, y in zip(o2, rec.axes): x.copy_(y, non_blocking=True)
    t7 = T()
    print(f"  dec: pageable H2D {t1-t0:.4f} staging memcpy {t2-t1:.4f} pinned H2D {t3-t2:.4f} decode {t4-t3:.4f} pageable D2H {t5-t4:.4f} pin alloc {t6-t5:.4f} pinned D2H {t7-t6:.4f}")
    del o, o2
