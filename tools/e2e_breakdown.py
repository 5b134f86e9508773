"""Where the host-buffer (e2e) compress / decompress time goes, per dataset.

Runs the bench workload's first dataset (280M particles x 3 f32, REL 1e-3)
and times each stage with a synchronize on both sides: H2D of the pinned
axes, compress_device, D2H of the container into the pinned stage, the bytes
materialization; then the decompress side the same way.  Experiments only.
"""

import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_10305_b200 as gz  # noqa: E402
from paper_2508_10305_b200 import pipeline as P  # noqa: E402


def t_(f, reps=3):
    best = 1e9
    out = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3, out


def main():
    torch.cuda.set_device(0)
    pos, vel = bench.gen_hacc(bench.PARTICLES, 280, torch.device("cuda"))
    cfg = gz.CompressConfig(error_bound=1e-3)
    for name, axes in (("pos", pos), ("vel", vel)):
        host = [a.cpu().pin_memory() for a in axes]
        nbytes = sum(a.numel() * 4 for a in host)
        hds = gz.Dataset.from_axes(host)
        ms_e2e, blob = t_(lambda: gz.compress(hds, cfg))
        ms_h2d, dev = t_(lambda: [a.to("cuda", non_blocking=True) for a in host])
        dds = gz.Dataset.from_axes(dev)
        ms_cd, cont = t_(lambda: P.compress_device(dds, cfg))
        n = cont.numel()
        ms_d2h, _ = t_(lambda: P._pinned(n)[:n].copy_(cont))
        ms_bytes, _ = t_(lambda: P._device_to_bytes(cont))
        print(f"{name} compress: e2e {ms_e2e:.2f} ms ({nbytes / ms_e2e / 1e6:.1f} GB/s) | H2D {ms_h2d:.2f} "
              f"({nbytes / ms_h2d / 1e6:.1f} GB/s) | compress_device {ms_cd:.2f} | D2H container {ms_d2h:.2f} "
              f"({n / ms_d2h / 1e6:.1f} GB/s, {n / 1e6:.0f} MB) | _device_to_bytes {ms_bytes:.2f}")
        ms_de2e, _ = t_(lambda: gz.decompress(blob))
        ms_tdb, (t, h) = t_(lambda: P._to_device_bytes(blob))
        host_b = P._host_bytes(blob)
        stage = P._pinned(host_b.size)[: host_b.size]
        ms_mm, _ = t_(lambda: P._par_memmove(stage.data_ptr(), host_b.ctypes.data, host_b.size))
        ms_h2, _ = t_(lambda: t.copy_(stage, non_blocking=True))
        cr = torch.cuda.cudart()
        ptr, sz = host_b.ctypes.data, host_b.size

        def reg():
            assert int(cr.cudaHostRegister(ptr, sz, 0)) == 0
        ms_reg, _ = t_(lambda: (reg(), cr.cudaHostUnregister(ptr)), reps=2)
        reg()
        src = torch.from_numpy(host_b)
        ms_h2r, _ = t_(lambda: t.copy_(src, non_blocking=True))
        cr.cudaHostUnregister(ptr)
        ms_page, _ = t_(lambda: t.copy_(src, non_blocking=False))
        fresh = lambda: P._api.PyBytes_FromStringAndSize(None, sz)  # noqa: E731

        def reg_fresh():
            b = fresh()
            a = P.ctypes.cast(P.ctypes.c_char_p(b), P.ctypes.c_void_p).value
            assert int(cr.cudaHostRegister(a, sz, 0)) == 0
            cr.cudaHostUnregister(a)
        ms_regf, _ = t_(reg_fresh, reps=2)
        print(f"  register+unregister {ms_reg:.2f} | H2D from registered bytes {ms_h2r:.2f} | pageable H2D {ms_page:.2f}"
              f" | fresh bytes register+unregister {ms_regf:.2f}")
        print(f"  bytes->pinned memmove {ms_mm:.2f} ({host_b.size / ms_mm / 1e6:.1f} GB/s) | pinned->device {ms_h2:.2f}")
        ms_dd, ds = t_(lambda: P.decompress_device(t, header=h))
        outs = [torch.empty(a.numel(), dtype=a.dtype, pin_memory=True) for a in ds.axes]
        ms_out, _ = t_(lambda: [o.copy_(a, non_blocking=True) for o, a in zip(outs, ds.axes)])
        ms_alloc, _ = t_(lambda: [torch.empty(a.numel(), dtype=a.dtype, pin_memory=True) for a in ds.axes])
        print(f"{name} decompress: e2e {ms_de2e:.2f} ms ({nbytes / ms_de2e / 1e6:.1f} GB/s) | bytes->device "
              f"{ms_tdb:.2f} | decompress_device {ms_dd:.2f} | D2H axes {ms_out:.2f} "
              f"({nbytes / ms_out / 1e6:.1f} GB/s) | pinned alloc {ms_alloc:.2f}")
        del host, hds, dev, dds, cont, blob, t, ds, outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
