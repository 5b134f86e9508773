"""Parity of the CUDA path against the reference (golden fixtures) and the
CPU oracle, through the public API and the C ABI.  Needs a B200."""

import numpy as np
import pytest
import torch

from _golden import CASES, CONTAINERS, GOLDEN, case, case_ids, error_prefix, make_axes, sha
from oracle import gpz_oracle as O

pytestmark = pytest.mark.gpu

gz = pytest.importorskip("paper_2508_10305_b200")


def _cfg(eb, mode, bs, t, pres):
    return gz.CompressConfig(error_bound=eb, eb_mode=gz.EbMode(mode), block_size=bs, target_segs_per_axis=t,
                             preserve_order=pres)


def _outcome(fn):
    try:
        return fn(), None
    except gz.GpzError as exc:
        return None, (type(exc).__name__, error_prefix(str(exc)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.fixture(params=["default", "cta"])
def route(request, monkeypatch):
    """Encoder routing: the default (K2s / K2p for the blocks they take), or
    GPZB_ROUTE=cta, which sends every narrow block to the general CTA
    encoder K2 so that its sort paths stay pinned to the goldens too."""
    if request.param == "cta":
        monkeypatch.setenv("GPZB_ROUTE", "cta")
    return request.param


@pytest.mark.parametrize("name", case_ids())
def test_golden_case(name, route):
    (_, gen, count, dims, dt, eb, mode, bs, t, pres, seed, extra) = case(name)
    want = GOLDEN["cases"][name]
    axes = make_axes(gen, count, dims, dt, seed, extra, O)
    blob, err = _outcome(lambda: gz.compress(gz.Dataset.from_axes(axes), _cfg(eb, mode, bs, t, pres)))
    if want["error"]:
        assert err == (want["error"][0], error_prefix(want["error"][1]))
        return
    assert err is None, err
    assert len(blob) == want["container_len"]
    if blob != CONTAINERS[name]:
        ref = CONTAINERS[name]
        first = next(i for i in range(min(len(ref), len(blob))) if ref[i] != blob[i])
        raise AssertionError(f"{name}: first differing byte {first} of {len(ref)}")
    ds = gz.decompress(blob)
    assert sha(*ds.axes) == want["recon_sha"]


def test_device_tensors_and_numpy_give_same_bytes():
    axes = O.gen_clusters(50_000, dims=3, seed=3)
    cfg = gz.CompressConfig(error_bound=1e-3)
    a = gz.compress(gz.Dataset.from_axes(axes), cfg)
    b = gz.compress(gz.Dataset.from_axes([torch.from_numpy(x).cuda() for x in axes]), cfg)
    c = gz.compress_device(gz.Dataset.from_axes([torch.from_numpy(x) for x in axes]), cfg)
    assert a == b == bytes(c.cpu().numpy())
    assert a == O.compress(axes, O.Config(1e-3))


@pytest.mark.parametrize("seed", range(40))
def test_random_configs_against_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    dims = int(rng.integers(1, 4))
    dt = np.float32 if rng.random() < 0.7 else np.float64
    n = int(rng.integers(1, 6000))
    kind = int(rng.integers(0, 4))
    if kind == 0:
        axes = [rng.uniform(-5, 5, n).astype(dt) for _ in range(dims)]
    elif kind == 1:
        axes = [(rng.normal(0, 1, n) * 10 ** rng.uniform(-3, 3)).astype(dt) for _ in range(dims)]
    elif kind == 2:
        axes = [np.round(rng.uniform(0, 100, n), 1).astype(dt) for _ in range(dims)]
    else:
        axes = O.gen_clusters(n, dims=dims, seed=seed, prec=O.F32 if dt == np.float32 else O.F64,
                              sigma=float(10 ** rng.uniform(-4, -1)))
    eb = float(10 ** rng.uniform(-7, -1))
    mode = int(rng.integers(0, 2))
    bs = int(32 * rng.integers(1, 33))
    t = int(2 ** rng.integers(0, 8))
    pres = bool(rng.integers(0, 2))
    try:
        want, werr = O.compress(axes, O.Config(eb, mode, bs, t, pres)), None
    except O.OracleError as exc:
        want, werr = None, (type(exc).__name__, error_prefix(str(exc)))
    got, gerr = _outcome(lambda: gz.compress(gz.Dataset.from_axes(axes), _cfg(eb, mode, bs, t, pres)))
    assert gerr == werr
    if want is None:
        return
    assert got == want
    rec = gz.decompress(got)
    for x, y in zip(rec.axes, O.decompress(want)):
        assert np.array_equal(x, y)


def test_bitflip_outcomes_match_reference():
    g = GOLDEN["bitflip"]
    base = CONTAINERS["bitflip_base"]
    bad = []
    for pos, bit, cls, tag in g["outcomes"]:
        c = bytearray(base)
        c[pos] ^= 1 << bit
        ds, err = _outcome(lambda: gz.decompress(bytes(c)))
        got = ("ok", sha(*ds.axes)[:16]) if err is None else err
        if got != (cls, tag):
            bad.append((pos, bit, got, (cls, tag)))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:5]}"


def test_iter_blocks_matches_decompress_and_oracle():
    for name in ("clu3_f32_e3", "uni2_f64_pres", "clu3_bs96"):
        blob = CONTAINERS[name]
        parts = list(gz.iter_decompressed_blocks(blob))
        want = list(O.iter_blocks(blob))
        assert len(parts) == len(want)
        for p, w in zip(parts, want):
            for a, b in zip(p, w):
                assert np.array_equal(a, b)


def test_iter_blocks_stops_at_first_corrupt_block():
    blob = bytearray(CONTAINERS["clu3_bs96"])
    h = O.read_container(bytes(blob))
    # corrupt block 3's unique count so it exceeds its particle count
    start = 46 + 8 * (h[0].blocks + 1) + int(h[1][3])
    blob[start + 7] ^= 0x40
    got = []
    with pytest.raises(gz.CorruptData, match="block 3"):
        for b in gz.iter_decompressed_blocks(bytes(blob)):
            got.append(b)
    assert len(got) == 3


def test_million_particle_golden_fixture():
    big = GOLDEN["big"]
    axes = O.gen_clusters(1_000_000, dims=3, seed=42)
    ds = gz.Dataset.from_axes([torch.from_numpy(a).cuda() for a in axes])
    for eb in (1e-2, 1e-3, 1e-4):
        blob = gz.compress(ds, gz.CompressConfig(error_bound=eb))
        want = big[repr(eb)]
        assert (len(blob), sha(blob)) == (want["container_len"], want["container_sha"])
        assert sha(*gz.decompress(blob).axes) == want["recon_sha"]


def test_resolve_absolute_bound_matches_oracle():
    axes = O.gen_clusters(100_000, dims=3, seed=5)
    for mode in (0, 1):
        cfg = gz.CompressConfig(error_bound=1e-3, eb_mode=gz.EbMode(mode))
        assert gz.resolve_absolute_bound(gz.Dataset.from_axes(axes), cfg) == \
            O.absolute_bound(axes, O.Config(1e-3, mode))
    with pytest.raises(gz.DomainError, match="axis 0"):
        bad = [a.copy() for a in axes]
        bad[0][5] = np.inf
        gz.resolve_absolute_bound(gz.Dataset.from_axes(bad), gz.CompressConfig(error_bound=1e-3))


def test_nonfinite_abs_mode_detected_on_device():
    axes = [np.linspace(0, 1, 5000, dtype=np.float32) for _ in range(3)]
    axes[2][4000] = np.nan
    with pytest.raises(gz.DomainError, match="axis 2 contains non-finite"):
        gz.compress(gz.Dataset.from_axes(axes), gz.CompressConfig(1e-3, eb_mode=gz.EbMode.ABSOLUTE))


def test_sort_paths_are_all_exercised(monkeypatch):
    """Every offset-order path of K2 (GPZB_ROUTE=cta) and K2s (default
    routing) runs on the golden cases (K2s's general-offset mode:
    test_parity_extra_gpu.test_small_encoder_general_offsets)."""
    seen = {"cta": np.zeros(8, np.int64), "default": np.zeros(8, np.int64)}
    for route in ("cta", "default"):
        if route == "cta":
            monkeypatch.setenv("GPZB_ROUTE", "cta")
        else:
            monkeypatch.delenv("GPZB_ROUTE", raising=False)
        for name in case_ids():
            (_, gen, count, dims, dt, eb, mode, bs, t, pres, seed, extra) = case(name)
            if GOLDEN["cases"][name]["error"] or count == 0:
                continue
            axes = make_axes(gen, count, dims, dt, seed, extra, O)
            gz.compress_device(gz.Dataset.from_axes(axes), _cfg(eb, mode, bs, t, pres))
            seen[route] += np.array(gz.pipeline.last_path_counts())
    assert (seen["cta"][:5] > 0).all(), seen
    assert seen["default"][6] > 0, seen


def test_unsupported_block_size_is_loud():
    """Above 2^24 particles per block the library refuses (the workspace
    slices of K2b / K4b would not fit); the reference has no limit."""
    with pytest.raises(NotImplementedError):
        gz.compress(gz.Dataset.from_axes([np.zeros(64, np.float32)]), gz.CompressConfig(1e-3, block_size=1 << 25))


BIG_CASES = [  # (kind, dims, dtype, eb, mode, block_size, target, preserve_order, n)
    ("clusters", 3, np.float32, 1e-3, 1, 2048, 32, False, 5 * 2048 + 77),
    ("clusters", 3, np.float32, 1e-4, 1, 4096, 32, True, 3 * 4096 + 1),
    ("uniform", 2, np.float64, 1e-5, 1, 1056, 16, False, 4 * 1056 + 1055),
    ("lattice", 1, np.float32, 1e-4, 0, 8192, 64, True, 2 * 8192 + 5),
    ("uniform", 3, np.float32, 1e-7, 1, 2048, 32, False, 2048 + 3),  # half-bound axes / wide keys
    ("clusters", 2, np.float64, 1e-9, 1, 65536, 32, False, 65536 + 999),
    ("uniform", 3, np.float64, 1e-6, 1, 2048, 16, True, 3 * 2048 + 7),  # F64 + rank stream
    ("clusters", 3, np.float32, 1e-12, 0, 4096, 32, False, 4096 + 5),  # WidthOverflow (oracle: error)
]


@pytest.mark.parametrize("case_", BIG_CASES, ids=lambda c: f"{c[0]}{c[1]}_{np.dtype(c[2]).name}_bs{c[5]}")
def test_block_size_above_1024(case_):
    """block_size > 1024 (any positive multiple of 32, model.py:118-119):
    K2b / K4b give the oracle's container, errors and reconstruction, also
    through iter_decompressed_blocks and the chunked host decode."""
    kind, dims, dt, eb, mode, bs, t, pres, n = case_
    gen = {"clusters": O.gen_clusters, "uniform": O.gen_uniform, "lattice": O.gen_lattice}[kind]
    axes = gen(n, dims=dims, seed=bs + n, prec=O.F64 if dt == np.float64 else O.F32)
    ocfg = O.Config(eb, mode, bs, t, pres)
    try:
        want, werr = O.compress(axes, ocfg), None
    except O.OracleError as exc:
        want, werr = None, (type(exc).__name__, error_prefix(str(exc)))
    got, gerr = _outcome(lambda: gz.compress(gz.Dataset.from_axes(axes), _cfg(eb, mode, bs, t, pres)))
    assert gerr == werr
    if werr:
        return
    assert got == want
    rec = gz.decompress(got)
    for x, y in zip(rec.axes, O.decompress(want)):
        assert np.array_equal(x, y)
    blocks = list(gz.iter_decompressed_blocks(got))
    assert len(blocks) == (n + bs - 1) // bs
    for a in range(dims):
        assert np.array_equal(np.concatenate([b[a] for b in blocks]), rec.axes[a])


def test_block_size_above_1024_streamed_decode():
    """A > 32 MiB host container of 4096-particle blocks takes the chunked
    host decode (block ranges through K4b); values equal the one-shot device
    decode's, and the container equals the oracle's on sampled blocks."""
    n = 40 * 1024 * 1024 + 123
    g = torch.Generator(device="cuda").manual_seed(3)
    pts = torch.rand(n, 3, device="cuda", dtype=torch.float64, generator=g)
    axes = [pts[:, a].float().contiguous() for a in range(3)]
    del pts
    cfg = gz.CompressConfig(error_bound=1e-5, block_size=4096)
    c = gz.compress_device(gz.Dataset.from_axes(axes), cfg)
    blob = bytes(c.cpu().numpy())
    assert len(blob) >= 32 << 20
    host = gz.decompress(blob)
    dev = gz.decompress_device(c)
    for x, y in zip(host.axes, dev.axes):
        assert np.array_equal(x, y.cpu().numpy())
    h, table, payload = O.read_container(blob)
    glob_eb = h.eb_abs  # the dataset's resolved bound, as the container records it
    rng = np.random.default_rng(1)
    nb = (n + 4095) // 4096
    for b in list(rng.integers(0, nb, 12)) + [0, nb - 1]:
        lo, hi = int(b) * 4096, min((int(b) + 1) * 4096, n)
        want = O.encode_block([a[lo:hi].cpu().numpy() for a in axes], glob_eb, O.Config(1e-5, block_size=4096),
                              O.F32)
        assert bytes(payload[table[b]:table[b + 1]]) == want, int(b)


def test_block_size_above_1024_corruption():
    """Bit flips in a container of 2048-particle blocks: the error class and
    block of the oracle's decoder (pipeline.py:160-205), flip by flip."""
    axes = O.gen_clusters(3 * 2048 + 100, dims=3, seed=9)
    blob = O.compress(axes, O.Config(1e-3, block_size=2048))
    rng = np.random.default_rng(5)
    for bit in rng.choice(len(blob) * 8, size=300, replace=False):
        bad = bytearray(blob)
        bad[bit // 8] ^= 1 << (bit % 8)
        bad = bytes(bad)
        try:
            O.decompress(bad)
            werr = None
        except O.OracleError as exc:
            werr = (type(exc).__name__, error_prefix(str(exc)))
        gerr = _outcome(lambda: gz.decompress(bad))[1]
        assert gerr == werr, int(bit)


def test_large_sampled_block_parity():
    """50M particles: sampled blocks of the GPU container against the oracle's
    per-block encoder, and sampled decoded blocks against its decoder."""
    n = 50_000_000
    g = torch.Generator(device="cuda").manual_seed(11)
    centers = torch.rand(4096, 3, device="cuda", dtype=torch.float64, generator=g)
    assign = torch.arange(n, device="cuda") // (n // 4096 + 1)
    pts = centers[assign] + 0.002 * torch.randn(n, 3, device="cuda", dtype=torch.float64, generator=g)
    axes = [pts[:, a].float().contiguous() for a in range(3)]
    del pts, assign
    cfg = gz.CompressConfig(error_bound=1e-3)
    ds = gz.Dataset.from_axes(axes)
    c = gz.compress_device(ds, cfg)
    blob_head = c[:46].cpu().numpy().tobytes()
    nb = (n + 1023) // 1024
    table = c[46: 46 + 8 * (nb + 1)].cpu().numpy().view("<u8")
    pay0 = 46 + 8 * (nb + 1)
    assert int(table[-1]) + pay0 == c.numel()
    eb_abs = float(np.frombuffer(blob_head[18:26], "<f8")[0])
    assert eb_abs == gz.resolve_absolute_bound(ds, cfg)
    rec = gz.decompress_device(c)
    rng = np.random.default_rng(0)
    picks = sorted(set(rng.integers(0, nb, 300).tolist()) | {0, nb - 1})
    host_c = None
    for i in picks:
        sl = slice(i * 1024, min((i + 1) * 1024, n))
        block = [a[sl].cpu().numpy() for a in axes]
        want = O.encode_block(block, eb_abs, O.Config(1e-3), O.F32)
        got = c[pay0 + int(table[i]): pay0 + int(table[i + 1])].cpu().numpy().tobytes()
        assert got == want, f"block {i}"
        h = O.Header(3, O.F32, False, 1, 1e-3, eb_abs, 1024, n, nb)
        dec = O.decode_block(want, h)
        for a in range(3):
            assert np.array_equal(rec.axes[a][sl].cpu().numpy(), dec[a]), f"decode block {i}"
    del host_c


@pytest.mark.parametrize("kind", ["clusters", "velocity"])
def test_bitflips_on_warp_decoded_blocks(kind):
    """Full 1024-particle blocks take the warp decoder (K4w); the golden bit-flip
    container above is too small for it.  Seeded single-bit flips over the
    table and the payloads (every bit of each block's first 64 payload bytes +
    random ones): error class and "block i" prefix, or the reconstruction,
    must equal the oracle's (pinned to the reference)."""
    rng = np.random.default_rng(7 if kind == "clusters" else 8)
    if kind == "clusters":
        axes = O.gen_clusters(4096, dims=3, seed=31)
    else:  # offsets present: bulk motion + per-particle spread
        bulk = rng.normal(0, 0.3, size=(4, 3))
        axes = [(np.repeat(bulk[:, a], 1024) + rng.normal(0, 0.05, 4096)).astype(np.float32) for a in range(3)]
    blob = O.compress(axes, O.Config(1e-3))
    assert gz.compress(gz.Dataset.from_axes(axes), gz.CompressConfig(1e-3)) == blob
    h, table, _ = O.read_container(blob)
    base = 46 + 8 * (h.blocks + 1)
    positions = set()
    for i in range(h.blocks):
        s = base + int(table[i])
        positions.update(range(s, min(s + 64, base + int(table[i + 1]))))
    positions.update(rng.integers(46, len(blob), 600).tolist())
    bad = []
    for pos in sorted(positions):
        for bit in range(8):
            c = bytearray(blob)
            c[pos] ^= 1 << bit
            ds, err = _outcome(lambda: gz.decompress(bytes(c)))
            try:
                want = ("ok", sha(*O.decompress(bytes(c))))
            except O.OracleError as exc:
                want = (type(exc).__name__, error_prefix(str(exc)))
            got = ("ok", sha(*ds.axes)) if err is None else err
            if got != want:
                bad.append((pos, bit, got, want))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:5]}"


def test_batched_calls_match_single_calls():
    """compress_batch_device / decompress_batch_device (one stream + workspace
    per dataset) give the bytes and values of the one-at-a-time calls."""
    sets = [O.gen_clusters(300_000, dims=3, seed=s) for s in (1, 2)] + [O.gen_uniform(70_001, dims=2, seed=3)]
    cfg = gz.CompressConfig(error_bound=1e-3)
    dss = [gz.Dataset.from_axes([torch.from_numpy(a).cuda() for a in axes]) for axes in sets]
    batch = gz.compress_batch_device(dss, cfg)
    for ds, c in zip(dss, batch):
        assert torch.equal(c, gz.compress_device(ds, cfg))
    recs = gz.decompress_batch_device(batch)
    for c, r in zip(batch, recs):
        want = gz.decompress_device(c)
        assert all(torch.equal(x, y) for x, y in zip(r.axes, want.axes))


@pytest.mark.parametrize("prec,dims", [(O.F32, 3), (O.F64, 3), (O.F64, 2), (O.F32, 1)])
def test_offset_free_warp_blocks(prec, dims):
    """Full blocks with no offset stream (every log2 m = 0) and few runs take
    K4w's run-values body (each run's reconstruction computed once); the
    result must be the oracle's, bit for bit, in every precision."""
    rng = np.random.default_rng(40 + dims)
    dt = np.float64 if prec == O.F64 else np.float32
    centers = rng.uniform(0, 1, size=(8, dims))  # one tight cluster per block: Q_a <= t, so log2 m = 0
    axes = [(np.repeat(centers[:, a], 1024) + rng.normal(0, 0.001, 8192)).astype(dt) for a in range(dims)]
    blob = O.compress(axes, O.Config(1e-3))
    h, table, _ = O.read_container(blob)
    assert gz.compress(gz.Dataset.from_axes(axes), gz.CompressConfig(1e-3)) == blob
    rec = gz.decompress(blob)
    for x, y in zip(rec.axes, O.decompress(blob)):
        assert np.array_equal(x, y)
    # the case is what it claims: no offsets, few runs
    base = 46 + 8 * (h.blocks + 1)
    for i in range(h.blocks):
        blk = blob[base + int(table[i]): base + int(table[i + 1])]
        S = 8 if prec == O.F64 else 4
        wpos = 8 + dims * (2 * S + 5)
        assert blk[wpos + 2] == 0  # w_off
        assert int.from_bytes(blk[4:8], "little") <= (128 if prec == O.F64 else 256)


@pytest.mark.parametrize("mode,pres,prec", [(1, False, O.F32), (0, True, O.F64)])
def test_remembered_header_matches_container(mode, pres, prec):
    """compress_device attaches the parsed global header to its result (so a
    device decode skips the header read); it must equal the header parsed
    from the container bytes, and an in-place change of the tensor must make
    decompress read the bytes again."""
    axes = O.gen_clusters(20_000, dims=3, seed=4, prec=prec)
    ds = gz.Dataset.from_axes([torch.from_numpy(a).cuda() for a in axes])
    c = gz.compress_device(ds, _cfg(1e-3, mode, 1024, 32, pres))
    h1 = gz.pipeline._known_header(c)
    h2 = gz.pipeline.parse_header(c[:46].cpu().numpy().tobytes(), c.numel())
    assert h1 is not None
    assert all(getattr(h1, f) == getattr(h2, f) for f, _ in type(h1)._fields_)
    c[4] ^= 0xFF  # the version field: the container is now invalid
    assert gz.pipeline._known_header(c) is None
    with pytest.raises(gz.CorruptData):
        gz.decompress_device(c)
