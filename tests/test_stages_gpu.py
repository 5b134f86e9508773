"""Per-stage parity of the device stage entry points against the oracle
(quantizer.derive_geometry / quantize_block, container.compact) and the
reference's code fixed point (/root/reference/pkg/tests/test_pipeline.py:75-88).
Needs a B200."""

import numpy as np
import pytest
import torch

from oracle import gpz_oracle as O

pytestmark = pytest.mark.gpu

gz = pytest.importorskip("paper_2508_10305_b200")
from paper_2508_10305_b200 import stages  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


CONFIGS = [
    ("clusters", 3, np.float32, 1e-3, 1024, 32),
    ("uniform", 2, np.float64, 1e-5, 512, 16),
    ("lattice", 1, np.float32, 1e-4, 256, 32),
    ("clusters", 3, np.float64, 1e-8, 1024, 64),  # 64-bit keys (1e-9 overflows, like the oracle)
    ("uniform", 2, np.float32, 1e-8, 1024, 32),  # half-bound axes (the edge-snap quantizer); 3D overflows
]


def _axes(kind, dims, dt, n, seed):
    gen = {"clusters": O.gen_clusters, "uniform": O.gen_uniform, "lattice": O.gen_lattice}[kind]
    return gen(n, dims=dims, seed=seed, prec=O.F64 if dt == np.float64 else O.F32)


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: f"{c[0]}{c[1]}_{np.dtype(c[2]).name}_{c[3]}")
def test_geometry_and_codes_match_oracle(cfg):
    kind, dims, dt, eb, bs, t = cfg
    n = 50 * bs + bs // 2  # a partial tail block
    axes = _axes(kind, dims, dt, n, 3)
    prec = O.F64 if dt == np.float64 else O.F32
    eb_abs = O.absolute_bound(axes, O.Config(eb))
    ds = gz.Dataset.from_axes(axes)
    geo = stages.block_geometry(ds, eb_abs, bs, t)
    seg, off = stages.quantize(ds, eb_abs, bs, t)
    lohi, Q, N, bits = (geo[k].cpu().numpy() for k in ("lohi", "Q", "N", "log2m"))
    seg = seg.cpu().numpy().view(np.uint64)
    off = off.cpu().numpy().view(np.uint64)
    for b in range(len(Q)):
        sl = slice(b * bs, min((b + 1) * bs, n))
        blk = [a[sl] for a in axes]
        mins = [float(a.min()) for a in blk]
        maxs = [float(a.max()) for a in blk]
        g = O.geometry(mins, maxs, eb_abs, t, prec)
        assert lohi[b, :, 0].tolist() == mins and lohi[b, :, 1].tolist() == maxs, b
        assert Q[b].tolist() == list(g.Q) and N[b].tolist() == list(g.N), b
        assert bits[b].tolist() == list(g.bits), b
        qs = [O.quantize_axis(blk[a], mins[a], maxs[a], g.Q[a], eb_abs, prec) for a in range(dims)]
        ws, wo = O.linearize(qs, g)
        assert np.array_equal(seg[sl], ws) and np.array_equal(off[sl], wo), b


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: f"{c[0]}{c[1]}_{np.dtype(c[2]).name}_{c[3]}")
@pytest.mark.parametrize("pres", [False, True])
def test_encode_payloads_match_encode_block(cfg, pres):
    """gpzb_encode_payloads: every block's payload equals the oracle's
    _encode_block(slice, eb_abs, cfg, prec) (pipeline.py:38-70) byte for
    byte, offsets included, at an absolute bound that is not the dataset's
    own resolved one."""
    kind, dims, dt, eb, bs, t = cfg
    n = 20 * bs + bs // 3
    axes = _axes(kind, dims, dt, n, 11)
    prec = O.F64 if dt == np.float64 else O.F32
    eb_abs = O.absolute_bound(axes, O.Config(eb)) * 1.37
    ocfg = O.Config(eb, block_size=bs, target_segs_per_axis=t, preserve_order=pres)
    try:
        want = [O.encode_block([a[b * bs:(b + 1) * bs] for a in axes], eb_abs, ocfg, prec)
                for b in range((n + bs - 1) // bs)]
    except O.WidthOverflow:
        with pytest.raises(gz.WidthOverflow):
            stages.encode_payloads(gz.Dataset.from_axes(axes), eb_abs, bs, t, pres)
        return
    pay, offs = stages.encode_payloads(gz.Dataset.from_axes(axes), eb_abs, bs, t, pres)
    offs = offs.cpu().numpy()
    assert offs[0] == 0 and offs[-1] == pay.numel() == sum(len(w) for w in want)
    got = bytes(pay.cpu().numpy())
    for b, w in enumerate(want):
        assert got[offs[b]:offs[b + 1]] == w, b


def test_geometry_errors_match_oracle():
    # a block whose range over the bound needs more than 64-bit bin indices
    axes = [np.concatenate([np.zeros(1024), np.array([0.0, 1e300])]).astype(np.float64)]
    ds = gz.Dataset.from_axes(axes)
    with pytest.raises(gz.WidthOverflow, match="block 1"):
        stages.block_geometry(ds, 1e-300, 1024, 32)
    with pytest.raises(gz.DomainError):
        stages.quantize(ds, -1.0, 1024, 32)
    bad = [np.array([0.0, np.nan, 1.0])]
    with pytest.raises(gz.DomainError, match="axis 0 contains non-finite"):
        stages.quantize(gz.Dataset.from_axes(bad), 0.1, 1024, 32)


def test_quantized_code_fixed_point_with_carried_geometry():
    """/root/reference/pkg/tests/test_pipeline.py:75-88 on the device: the
    codes of the reconstruction, quantized with the original blocks'
    geometry, equal the original codes (per block, in (seg, off) order)."""
    rng = np.random.default_rng(3)
    axes = [rng.uniform(0, 1, 2048) for _ in range(2)]  # 2D float64
    eb_abs = 0.01
    cfg = gz.CompressConfig(error_bound=eb_abs, eb_mode=gz.EbMode.ABSOLUTE)
    ds = gz.Dataset.from_axes(axes)
    rec = gz.decompress(gz.compress(ds, cfg))
    lohi = stages.block_geometry(ds, eb_abs)["lohi"]
    s0, o0 = (t.cpu().numpy().view(np.uint64) for t in stages.quantize(ds, eb_abs))
    s1, o1 = (t.cpu().numpy().view(np.uint64) for t in stages.quantize(rec, eb_abs, lohi=lohi))
    for b in range(2):
        sl = slice(b * 1024, (b + 1) * 1024)
        k0 = np.lexsort((o0[sl], s0[sl]))
        k1 = np.lexsort((o1[sl], s1[sl]))
        assert np.array_equal(s0[sl][k0], s1[sl][k1]) and np.array_equal(o0[sl][k0], o1[sl][k1]), b


@pytest.mark.parametrize("nb", [0, 1, 7, 8192, 8193, 100_003])
def test_scan_sizes_matches_compact(nb):
    rng = np.random.default_rng(nb)
    sizes = rng.integers(0, 5000, nb).astype(np.int64)
    got = stages.scan_sizes(torch.from_numpy(sizes)).cpu().numpy()
    want = np.zeros(nb + 1, np.int64)
    want[1:] = np.cumsum(sizes)
    assert np.array_equal(got, want)
