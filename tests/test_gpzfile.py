""".gpz files and block-range access (gpzfile.py).

CPU: the host step (table slice -> self-contained sub-container) checked with
the oracle decoder against the full container.  GPU: decompress_blocks from
bytes, CUDA tensors and files; error block numbering; file round trips.
"""

import numpy as np
import pytest

from oracle import gpz_oracle as O

gz = pytest.importorskip("paper_2508_10305_b200")
from paper_2508_10305_b200 import gpzfile as F  # noqa: E402


def _blob(n=10_000, seed=3, bs=1024):
    axes = O.gen_clusters(n, dims=3, seed=seed)
    return axes, O.compress(axes, O.Config(1e-3, block_size=bs))


@pytest.mark.parametrize("first,last", [(0, 10), (0, 1), (3, 7), (9, 10), (4, 4)])
def test_sub_container_decodes_like_the_full_container(first, last, tmp_path):
    axes, blob = _blob()
    full = O.decompress(blob)
    for src in (blob, str(tmp_path / "c.gpz")):
        if not isinstance(src, bytes):
            with open(src, "wb") as f:
                f.write(blob)
        head, t, pay = F._read_range(src, first, last)
        sub = F.sub_container(head, t, pay, first, last)
        got = O.decompress(sub) if last > first else [np.empty(0, np.float32)] * 3
        lo, hi = first * 1024, min(last * 1024, 10_000)
        for a, b in zip(got, full):
            assert np.array_equal(a, b[lo:hi])


def test_block_range_checks():
    _, blob = _blob()
    with pytest.raises(IndexError):
        F._read_range(blob, 5, 11)
    with pytest.raises(gz.CorruptData):
        F._read_range(blob[:60], 0, 10)


def test_write_read_container_bytes(tmp_path):
    _, blob = _blob()
    p = tmp_path / "x.gpz"
    assert F.write_container(p, blob) == len(blob)
    assert F.read_container(p) == blob


gpu = pytest.mark.gpu


def _torch():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@gpu
def test_decompress_blocks_all_sources(tmp_path):
    torch = _torch()
    axes = O.gen_clusters(300_000, dims=3, seed=8)
    ds = gz.Dataset.from_axes(axes)
    cfg = gz.CompressConfig(error_bound=1e-3)
    dev = gz.compress_device(ds, cfg)
    blob = bytes(dev.cpu().numpy())
    path = tmp_path / "c.gpz"
    assert F.write_container(path, dev) == len(blob)
    assert F.read_container(path) == blob
    assert torch.equal(F.read_container(path, device=True), dev)
    full = gz.decompress(blob)
    nb = (300_000 + 1023) // 1024
    for first, last in [(0, nb), (0, 1), (17, 90), (nb - 1, nb), (100, 100)]:
        lo, hi = first * 1024, min(last * 1024, 300_000)
        for src in (blob, dev, str(path)):
            got = F.decompress_blocks(src, first, last)
            for a, b in zip(got.axes, full.axes):
                assert np.array_equal(a, b[lo:hi])
    seen = 0
    for first, part in F.iter_file_blocks(str(path), chunk_blocks=50):
        assert first == seen * 50
        lo = first * 1024
        assert np.array_equal(part.axes[2], full.axes[2][lo:lo + part.count])
        seen += 1
    assert seen == (nb + 49) // 50


@gpu
def test_decompress_blocks_error_names_original_block():
    _torch()
    axes, blob = _blob(20_000, seed=4)
    h, table, _ = O.read_container(blob)
    bad = bytearray(blob)
    base = 46 + 8 * (h.blocks + 1)
    bad[base + int(table[12]) + 4] ^= 0xFF  # block 12's unique-id count
    with pytest.raises(gz.CorruptData, match=r"^block 12: "):
        F.decompress_blocks(bytes(bad), 10, 15)
    F.decompress_blocks(bytes(bad), 13, 19)  # blocks after the corrupt one decode
