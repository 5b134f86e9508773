"""Pin the CPU oracle against the reference's own outputs (CPU only).

The golden fixtures were produced by the reference package itself
(tests/golden/make_golden.py); the oracle must reproduce every container,
reconstruction and error outcome, plus the reference's published known
answers (tests/test_codec.py:98-106, tests/test_acceptance.py:180-184)."""

import numpy as np
import pytest

from _golden import CASES, CONTAINERS, GOLDEN, case, case_ids, error_prefix, make_axes, sha
from oracle import gpz_oracle as O


@pytest.mark.parametrize("name", case_ids())
def test_oracle_matches_reference_case(name):
    (_, gen, count, dims, dt, eb, mode, bs, t, pres, seed, extra) = case(name)
    want = GOLDEN["cases"][name]
    axes = make_axes(gen, count, dims, dt, seed, extra, O)
    assert sha(*axes) == want["input_sha"]
    if want["error"]:
        with pytest.raises(O.OracleError) as ei:
            O.compress(axes, O.Config(eb, mode, bs, t, pres))
        assert type(ei.value).__name__ == want["error"][0]
        assert str(ei.value) == want["error"][1]
        return
    blob = O.compress(axes, O.Config(eb, mode, bs, t, pres))
    assert len(blob) == want["container_len"]
    assert sha(blob) == want["container_sha"]
    assert blob == CONTAINERS[name]
    assert sha(*O.decompress(blob)) == want["recon_sha"]


def test_known_answer_four_particles():
    # [0.2,3.7,5.1,7.9] f64, ABS eb 0.5, bs 32 -> 96 bytes
    hexs = ("47505a31010001010000000000000000e03f000000000000e03f200000000400000000000000010000000000"
            "00000000000000000000220000000000000004000000040000009a9999999999c93f9a99999999991f4000080000"
            "00020100dc0f")
    blob = O.compress([np.array([0.2, 3.7, 5.1, 7.9])], O.Config(0.5, O.ABSOLUTE, 32))
    assert blob.hex() == hexs


def test_bit_layout_golden_bytes():
    # codec.py bit layout, tests/test_codec.py:98-106
    assert O.pack(np.array([1, 2, 1], np.uint64), 2) == bytes([0b00011001])
    assert O.pack(np.array([5], np.uint64), 3) == bytes([0b00000101])
    assert O.pack(np.zeros(3, np.uint64), 0) == b""
    assert O.unpack(bytes([0b00011001]), 3, 2).tolist() == [1, 2, 1]
    with pytest.raises(O.CorruptData):
        O.unpack(bytes([0b11011001]), 3, 2)  # dirty padding


def test_pack_roundtrip_all_widths():
    rng = np.random.default_rng(4242)
    for w in range(65):
        n = int(rng.integers(0, 70))
        v = rng.integers(0, 1 << min(w, 63), n, dtype=np.uint64) if w else np.zeros(n, np.uint64)
        if w == 64 and n:
            v[0] = np.uint64(2**64 - 1)
        raw = O.pack(v, w)
        assert len(raw) == (n * w + 7) // 8
        assert np.array_equal(O.unpack(raw, n, w), v)


def test_oracle_bitflip_outcomes_match_reference():
    g = GOLDEN["bitflip"]
    base = CONTAINERS["bitflip_base"]
    assert sha(base) == g["sha"]
    for pos, bit, cls, tag in g["outcomes"][::3]:
        c = bytearray(base)
        c[pos] ^= 1 << bit
        try:
            out = O.decompress(bytes(c))
            got = ("ok", sha(*out)[:16])
        except O.OracleError as exc:
            got = (type(exc).__name__, error_prefix(str(exc)))
        assert got == (cls, tag), (pos, bit)


def test_golden_million_particle_fixture():
    big = GOLDEN["big"]
    axes = O.gen_clusters(1_000_000, dims=3, seed=42)
    assert sha(*axes) == big["input_sha"]
    assert axes[0][:4].tobytes().hex() == "2cd0413f6e94433f272a453f5205483f"
    for eb in (1e-2, 1e-3, 1e-4):
        blob = O.compress(axes, O.Config(eb))
        want = big[repr(eb)]
        assert (len(blob), sha(blob)) == (want["container_len"], want["container_sha"])
    assert big[repr(1e-3)]["container_len"] == 1_550_113  # tests/test_acceptance.py:184


def test_iter_blocks_matches_decompress():
    blob = CONTAINERS["clu3_f32_e3"]
    full = O.decompress(blob)
    parts = list(O.iter_blocks(blob))
    for a in range(3):
        assert np.array_equal(np.concatenate([p[a] for p in parts]), full[a])


@pytest.mark.parametrize("kind", ["uniform", "lattice"])
def test_oracle_matches_reference_stress_fixtures(kind):
    """1M-particle UNIFORM_BOX / JITTERED_LATTICE (SURVEY.md §8d stress
    fixtures) at rel-eb 1e-2 / 1e-3 / 1e-4: container and reconstruction
    SHA-256 of the reference itself (tests/golden/make_golden_stress.py)."""
    from _golden import STRESS

    gen = {"uniform": O.gen_uniform, "lattice": O.gen_lattice}[kind]
    axes = gen(1_000_000, dims=3, seed=42)
    want = STRESS[kind]
    assert sha(*axes) == want["input_sha"]
    for eb in (1e-2, 1e-3, 1e-4):
        blob = O.compress(axes, O.Config(eb))
        assert (len(blob), sha(blob)) == (want[repr(eb)]["container_len"], want[repr(eb)]["container_sha"])
        assert sha(*O.decompress(blob)) == want[repr(eb)]["recon_sha"]
