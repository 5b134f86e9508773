"""BASELINE.json configurations beyond the bench workload, at full size.

configs[2]  LiDAR-style clustered point cloud, 500M points xyz f32, rel-eb 1e-4
configs[3]  decompression sweep over rel-eb 1e-2 / 1e-3 / 1e-4 on 1B particles

At these sizes the oracle cannot run end to end, so parity is checked by
(1) sampled blocks of the GPU container against the oracle's per-block
encoder and decoder (bit-exact bytes and values), (2) the size-independent
properties: the offset table is consistent with the container length, and
the whole reconstruction is within the bound under the reference's block
pairing (K5, metrics.verify_bound semantics), (3) compression ratio = input
bytes / container bytes with the container byte-exact per sampled block.
"""

import numpy as np
import pytest
import torch

from oracle import gpz_oracle as O

pytestmark = pytest.mark.gpu

gz = pytest.importorskip("paper_2508_10305_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def gen_lidar(n: int, seed: int):
    """bench.py's configs[2] generator (the benchmarked data is the tested data)."""
    import bench

    return bench.gen_lidar(n, seed, torch.device("cuda"))


def gen_clusters_dev(n: int, clusters: int, sigma: float, seed: int):
    """bench.py's configs[3] generator."""
    import bench

    return bench.gen_clusters(n, clusters, sigma, seed, torch.device("cuda"))


def sampled_parity(axes, cfg, container, rec, picks):
    n = axes[0].numel()
    bs = cfg.block_size
    nb = (n + bs - 1) // bs
    head = container[:46].cpu().numpy().tobytes()
    table = container[46: 46 + 8 * (nb + 1)].cpu().numpy().view("<u8")
    pay0 = 46 + 8 * (nb + 1)
    assert int(table[0]) == 0 and int(table[-1]) + pay0 == container.numel()
    eb_abs = float(np.frombuffer(head[18:26], "<f8")[0])
    oc = O.Config(cfg.error_bound, eb_mode=cfg.eb_mode.value, block_size=bs,
                  target_segs_per_axis=cfg.target_segs_per_axis)
    h = O.Header(3, O.F32, False, cfg.eb_mode.value, cfg.error_bound, eb_abs, bs, n, nb)
    for i in picks:
        sl = slice(i * bs, min((i + 1) * bs, n))
        block = [a[sl].cpu().numpy() for a in axes]
        want = O.encode_block(block, eb_abs, oc, O.F32)
        got = container[pay0 + int(table[i]): pay0 + int(table[i + 1])].cpu().numpy().tobytes()
        assert got == want, f"block {i}"
        dec = O.decode_block(want, h)
        for a in range(3):
            assert np.array_equal(rec.axes[a][sl].cpu().numpy(), dec[a]), f"decode block {i}"
    return eb_abs


def _picks(nb, k=200, seed=0):
    rng = np.random.default_rng(seed)
    return sorted(set(rng.integers(0, nb, k).tolist()) | {0, nb - 1})


def test_config2_lidar_500m_rel_1e4():
    n = 500_000_000
    axes = gen_lidar(n, 500)
    ds = gz.Dataset.from_axes(axes)
    cfg = gz.CompressConfig(error_bound=1e-4)
    c = gz.compress_device(ds, cfg)
    rec = gz.decompress_device(c)
    nb = (n + 1023) // 1024
    eb_abs = sampled_parity(axes, cfg, c, rec, _picks(nb))
    assert eb_abs == gz.resolve_absolute_bound(ds, cfg)
    rep = gz.verify_bound(ds, rec, eb_abs, cfg)
    assert rep.ok and rep.max_err <= eb_abs and rep.checked == 3 * n
    print(f"lidar 500M rel 1e-4: CR {ds.nbytes / c.numel():.3f}, max_err/eb {rep.max_err / eb_abs:.6f}")


def test_config3_decompression_sweep_1b():
    n = 1_000_000_000
    axes = gen_clusters_dev(n, 32768, 0.002, 1000)
    ds = gz.Dataset.from_axes(axes)
    nb = (n + 1023) // 1024
    for k, eb in enumerate((1e-2, 1e-3, 1e-4)):
        cfg = gz.CompressConfig(error_bound=eb)
        c = gz.compress_device(ds, cfg)
        rec = gz.decompress_device(c)
        eb_abs = sampled_parity(axes, cfg, c, rec, _picks(nb, 100, seed=k))
        rep = gz.verify_bound(ds, rec, eb_abs, cfg)
        assert rep.ok and rep.max_err <= eb_abs
        print(f"1B clusters rel {eb:g}: CR {ds.nbytes / c.numel():.3f}")
        del c, rec
        torch.cuda.empty_cache()


@pytest.mark.parametrize("dims,f64,pres,eb", [(3, True, False, 1e-6), (2, False, True, 1e-3), (1, False, False, 1e-5),
                                             (3, False, True, 1e-4)])
def test_other_layouts_at_scale(dims, f64, pres, eb):
    """20M particles: float64 inputs, 1D/2D, preserve_order (rank stream +
    general encoder/decoder) — sampled blocks against the oracle, the whole
    reconstruction under the bound (K5), and order preservation."""
    n = 20_000_000
    g = torch.Generator(device="cuda").manual_seed(77 + dims)
    dt = torch.float64 if f64 else torch.float32
    c = torch.rand(2048, dims, generator=g, device="cuda", dtype=torch.float64)
    assign = torch.arange(n, device="cuda") * 2048 // n
    axes = [(c[assign, a] + 0.003 * torch.randn(n, generator=g, device="cuda", dtype=torch.float64)).to(dt)
            for a in range(dims)]
    del assign
    cfg = gz.CompressConfig(error_bound=eb, preserve_order=pres)
    ds = gz.Dataset.from_axes(axes)
    cont = gz.compress_device(ds, cfg)
    rec = gz.decompress_device(cont)
    nb = (n + 1023) // 1024
    head = cont[:46].cpu().numpy().tobytes()
    table = cont[46: 46 + 8 * (nb + 1)].cpu().numpy().view("<u8")
    pay0 = 46 + 8 * (nb + 1)
    eb_abs = float(np.frombuffer(head[18:26], "<f8")[0])
    prec = O.F64 if f64 else O.F32
    oc = O.Config(eb, block_size=1024, preserve_order=pres)
    h = O.Header(dims, prec, pres, 1, eb, eb_abs, 1024, n, nb)
    for i in _picks(nb, 60, seed=dims):
        sl = slice(i * 1024, min((i + 1) * 1024, n))
        block = [a[sl].cpu().numpy() for a in axes]
        want = O.encode_block(block, eb_abs, oc, prec)
        got = cont[pay0 + int(table[i]): pay0 + int(table[i + 1])].cpu().numpy().tobytes()
        assert got == want, f"block {i}"
        dec = O.decode_block(want, h)
        for a in range(dims):
            assert np.array_equal(rec.axes[a][sl].cpu().numpy(), dec[a]), f"decode block {i}"
    if pres:  # particles come back in their original order, each within the bound
        for a in range(dims):
            err = (rec.axes[a].double() - axes[a].double()).abs().max().item()
            assert err <= eb_abs
    rep = gz.verify_bound(ds, rec, eb_abs, cfg)
    assert rep.ok and rep.max_err <= eb_abs
