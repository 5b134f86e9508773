"""Parity of the CUDA path on the benchmarked workload and the reference's
robustness edge cases (needs a B200).

* the exact bench.py workload (gen_hacc, configs[1]: 280M positions and
  velocities, rel-eb 1e-3) — sampled blocks byte-compared with the oracle's
  per-block encoder and decoder (SURVEY.md §8c protocol for N > 10M);
* the reference's 1M UNIFORM_BOX / JITTERED_LATTICE stress fixtures
  (tests/golden/stress.json, made by the reference itself);
* every truncation of a container and trailing bytes
  (/root/reference/pkg/tests/test_container.py:86-94, container.py:188-193),
  with the oracle's error class and block;
* mixed +-0.0 block bounds: the one documented divergence (numpy's min/max
  sign is layout dependent), pinned to the sign bit of the stored bound.
"""

import numpy as np
import pytest
import torch

from _golden import CONTAINERS, STRESS, error_prefix, sha
from oracle import gpz_oracle as O

pytestmark = pytest.mark.gpu

gz = pytest.importorskip("paper_2508_10305_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _outcome(fn):
    try:
        fn()
        return None
    except (gz.GpzError, O.OracleError) as exc:
        return type(exc).__name__, error_prefix(str(exc))


@pytest.mark.parametrize("kind", ["uniform", "lattice"])
def test_stress_fixtures_match_reference(kind):
    gen = {"uniform": O.gen_uniform, "lattice": O.gen_lattice}[kind]
    axes = gen(1_000_000, dims=3, seed=42)
    want = STRESS[kind]
    ds = gz.Dataset.from_axes([torch.from_numpy(a).cuda() for a in axes])
    for eb in (1e-2, 1e-3, 1e-4):
        blob = gz.compress(ds, gz.CompressConfig(error_bound=eb))
        w = want[repr(eb)]
        assert (len(blob), sha(blob)) == (w["container_len"], w["container_sha"]), (kind, eb)
        assert sha(*gz.decompress(blob).axes) == w["recon_sha"], (kind, eb)


def test_bench_workload_sampled_blocks():
    """bench.py's own input (gen_hacc, 280M particles x 2 datasets, the
    headline configuration): >= 4096 random blocks plus the first and last
    of each dataset equal the oracle's _encode_block bytes, the container's
    eb_abs equals the oracle's bound, and sampled blocks decode bit-exactly."""
    import bench

    n = bench.PARTICLES
    pos, vel = bench.gen_hacc(n, 280, torch.device("cuda"))
    cfg = gz.CompressConfig(error_bound=1e-3)
    nb = (n + 1023) // 1024
    rng = np.random.default_rng(280)
    for name, axes in (("pos", pos), ("vel", vel)):
        ds = gz.Dataset.from_axes(axes)
        c = gz.compress_device(ds, cfg)
        head = c[:46].cpu().numpy().tobytes()
        eb_abs = float(np.frombuffer(head[18:26], "<f8")[0])
        lo = min(float(a.min()) for a in axes)
        hi = max(float(a.max()) for a in axes)
        assert eb_abs == 1e-3 * (hi - lo), name  # model.py:194-199, same IEEE ops
        table = c[46: 46 + 8 * (nb + 1)].cpu().numpy().view("<u8").astype(np.int64)
        pay0 = 46 + 8 * (nb + 1)
        assert int(table[0]) == 0 and int(table[-1]) + pay0 == c.numel()
        picks = sorted(set(rng.integers(0, nb, 4096).tolist()) | {0, nb - 1})
        cpu = [a.cpu().numpy() for a in axes]
        host = c.cpu().numpy()
        h = O.Header(3, O.F32, False, 1, 1e-3, eb_abs, 1024, n, nb)
        rec = gz.decompress_device(c)
        for k, i in enumerate(picks):
            sl = slice(i * 1024, min((i + 1) * 1024, n))
            want = O.encode_block([a[sl] for a in cpu], eb_abs, O.Config(1e-3), O.F32)
            got = host[pay0 + table[i]: pay0 + table[i + 1]].tobytes()
            assert got == want, f"{name} block {i}"
            if k % 8 == 0 or i in (0, nb - 1):  # decode one in eight, and both ends
                dec = O.decode_block(want, h)
                for a in range(3):
                    assert np.array_equal(rec.axes[a][sl].cpu().numpy(), dec[a]), f"{name} block {i} axis {a}"
        del c, rec


def _small_container() -> bytes:
    return CONTAINERS["bitflip_base"]  # 2D f32, 3 blocks of 512 (made by the reference)


def test_every_truncation_is_corrupt_like_the_oracle():
    blob = _small_container()
    for cut in range(len(blob)):
        bad = blob[:cut]
        want = _outcome(lambda: O.decompress(bad))
        got = _outcome(lambda: gz.decompress(bad))
        assert want is not None and want[0] == "CorruptData", cut
        assert got == want, cut


@pytest.mark.parametrize("extra", [b"\x00", b"\x00" * 7, b"\xff" * 16, bytes(range(64))])
def test_trailing_bytes_are_corrupt_like_the_oracle(extra):
    blob = _small_container() + extra
    want = _outcome(lambda: O.decompress(blob))
    assert want is not None and want[0] == "CorruptData"
    assert _outcome(lambda: gz.decompress(blob)) == want
    dev = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda()
    assert _outcome(lambda: gz.decompress_device(dev)) == want


def test_mixed_signed_zero_bounds_pinned():
    """numpy's min/max of a block holding both -0.0 and +0.0 returns a
    layout-dependent sign; the kernels order -0.0 below +0.0.
    The two containers may differ only in the sign bit of a stored block
    bound; every geometry, stream and reconstructed value is identical, and
    the oracle decodes the CUDA container to the same values."""
    rng = np.random.default_rng(5)
    axes = [rng.uniform(-1, 1, 4096).astype(np.float32) for _ in range(3)]
    for a in axes:  # axis minima / maxima at signed zeros, both signs present
        a[a < 0] = -a[a < 0]
        a[::97] = 0.0
        a[5::97] = -0.0
    cfg = gz.CompressConfig(error_bound=1e-3)
    got = gz.compress(gz.Dataset.from_axes(axes), cfg)
    want = O.compress(axes, O.Config(1e-3))
    assert len(got) == len(want)
    diff = np.flatnonzero(np.frombuffer(got, np.uint8) != np.frombuffer(want, np.uint8))
    nb = 4
    pay0 = 46 + 8 * (nb + 1)
    table = np.frombuffer(want, "<u8", count=nb + 1, offset=46)
    for d in diff:
        blk = int(np.searchsorted(table, d - pay0, side="right")) - 1
        rel = d - pay0 - int(table[blk])
        # header: u32 n, u32 U, then per axis f32 min (+0), f32 max (+4), u8, u32 (13 bytes)
        assert rel >= 8 and (rel - 8) % 13 in (3, 7), (d, rel)  # the top byte of a stored bound
        assert got[d] ^ want[d] == 0x80  # its sign bit, nothing else
    for a, b, c in zip(gz.decompress(got).axes, O.decompress(want), O.decompress(got)):
        assert np.array_equal(a, b) and np.array_equal(b, c)


def test_concurrent_threads_get_their_own_results():
    """compress / decompress from several host threads at once, on distinct
    data (safe for concurrent calls): every thread's bytes and
    values equal the sequential results (per-thread workspaces, pinned
    buffers and side buffers, pipeline._tls)."""
    import threading

    sets = [O.gen_clusters(300_000 + 1000 * k, dims=3, seed=40 + k) for k in range(4)]
    cfg = gz.CompressConfig(error_bound=1e-3)
    want = [gz.compress(gz.Dataset.from_axes(a), cfg) for a in sets]
    want_dev = [gz.compress_device(gz.Dataset.from_axes([torch.from_numpy(x).cuda() for x in a]), cfg).cpu()
                for a in sets]
    errs = []

    def work(k):
        try:
            ds = gz.Dataset.from_axes(sets[k])
            dsd = gz.Dataset.from_axes([torch.from_numpy(x).cuda() for x in sets[k]])
            for _ in range(6):
                blob = gz.compress(ds, cfg)
                assert blob == want[k], k
                rec = gz.decompress(blob)
                ref = O.decompress(want[k])
                assert all(np.array_equal(a, b) for a, b in zip(rec.axes, ref)), k
                c = gz.compress_device(dsd, cfg)
                assert torch.equal(c.cpu(), want_dev[k]), k
        except Exception as exc:  # noqa: BLE001
            errs.append((k, repr(exc)))

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs


@pytest.mark.parametrize("eb", [3e-3, 1e-3, 3e-4, 1e-4, 3e-5])
def test_velocity_blocks_wide_offsets_ties_long_runs(eb):
    """Velocity-like blocks from Σ log2 m <= 4 (K2s) to well above (K2's
    offset-order paths), with repeated (segment, offset) pairs and a run of
    200 identical particles: the whole container equals the oracle's."""
    rng = np.random.default_rng(int(eb * 1e6))
    n = 64 * 1024
    bulk = np.repeat(rng.normal(0, 0.3, size=(64, 3)), 1024, axis=0)
    pts = bulk + rng.normal(0, 0.05, size=(n, 3)) * rng.uniform(0.2, 3.0, size=(64, 1)).repeat(1024, axis=0)
    pts[5 * 1024:5 * 1024 + 200] = pts[5 * 1024]            # one long run of identical particles
    pts[9 * 1024:10 * 1024:2] = pts[9 * 1024 + 1:10 * 1024:2]  # pairs of identical particles
    axes = [np.ascontiguousarray(pts[:, a]).astype(np.float32) for a in range(3)]
    want = O.compress(axes, O.Config(eb))
    got = gz.compress(gz.Dataset.from_axes(axes), gz.CompressConfig(error_bound=eb))
    assert got == want


@pytest.mark.parametrize("kind,eb,lanes", [("clusters", 1e-2, 8), ("lattice", 1e-2, 16), ("uniform", 1e-4, 32)])
def test_payload_copy_lane_groups_match_oracle(kind, eb, lanes):
    """K3b moves each payload with 8, 16 or 32 lanes by the container's
    average payload (< 384 B, < 1024 B, else): one dataset per group (their
    averages measured with the oracle: 95 B, 627 B, 4,155 B), the whole
    container and the reconstruction equal the oracle's (pipeline.py:73-103,
    container.py:211-230)."""
    gen = {"clusters": O.gen_clusters, "lattice": O.gen_lattice, "uniform": O.gen_uniform}[kind]
    n = 65536
    axes = gen(n, seed=3)
    want = O.compress(axes, O.Config(error_bound=eb))
    nb = n // 1024
    avg = (len(want) - 54 - 8 * (nb + 1)) / nb
    assert {8: avg < 384, 16: 384 <= avg < 1024, 32: avg >= 1024}[lanes], avg
    ds = gz.Dataset.from_axes([torch.from_numpy(a).cuda() for a in axes])
    blob = gz.compress(ds, gz.CompressConfig(error_bound=eb))
    assert blob == want
    got = gz.decompress(blob).axes
    for g, o in zip(got, O.decompress(want)):
        assert np.asarray(g).tobytes() == np.asarray(o).tobytes()
