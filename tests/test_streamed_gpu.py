"""The chunked host decompress (pipeline._decode_streamed): containers of 32
MiB and more are uploaded, decoded (gpzb_decompress_range_async, include/
gpzb.h) and downloaded chunk by chunk.  Its output and its errors must be
exactly those of the one-shot decode of the same container already on the
device (which test_gpu_parity.py pins to the oracle)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

gz = pytest.importorskip("paper_2508_10305_b200")
from paper_2508_10305_b200 import pipeline as P  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _noisy(n, dims, seed, f64=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    c = torch.randn(4096, dims, generator=g, device="cuda", dtype=torch.float64)
    assign = torch.arange(n, device="cuda") * 4096 // n
    dt = torch.float64 if f64 else torch.float32
    return [(c[assign, a] + 0.05 * torch.randn(n, generator=g, device="cuda", dtype=torch.float64)).to(dt).cpu()
            for a in range(dims)]


def _one_shot(blob):
    t = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda()
    return gz.decompress_device(t)


def _err(f):
    try:
        f()
    except Exception as e:  # noqa: BLE001
        return type(e).__name__, str(e)
    return None


@pytest.fixture(scope="module")
def blob():
    axes = _noisy(16_000_000, 3, 5)
    b = gz.compress(gz.Dataset.from_axes(axes), gz.CompressConfig(error_bound=1e-4))
    assert len(b) >= (32 << 20)
    return b


def test_streamed_matches_one_shot(blob):
    h = P.parse_header(blob[:46], len(blob))
    plan = P._streamed_plan(P._host_bytes(blob), h)
    assert plan is not None and len(plan[1]) >= 16
    got = gz.decompress(blob)
    want = _one_shot(blob)
    dev = gz.decompress_device(blob)
    for a in range(3):
        w = want.axes[a].cpu().numpy()
        assert np.array_equal(got.axes[a], w)
        assert np.array_equal(dev.axes[a].cpu().numpy(), w)


@pytest.mark.parametrize("dims,f64,pres", [(2, True, False), (3, False, True)])
def test_streamed_other_layouts(dims, f64, pres):
    axes = _noisy(12_000_000 if pres else 20_000_000, dims, 9 + dims, f64)
    cfg = gz.CompressConfig(error_bound=1e-6, preserve_order=pres)
    ds = gz.Dataset.from_axes(axes)
    b = gz.compress(ds, cfg)
    assert len(b) >= (32 << 20)
    got = gz.decompress(b)
    want = _one_shot(b)
    for a in range(dims):
        assert np.array_equal(got.axes[a], want.axes[a].cpu().numpy())
    if pres:  # original order, every particle within the bound
        eb_abs = gz.resolve_absolute_bound(ds, cfg)
        for a in range(dims):
            assert np.abs(got.axes[a].astype(np.float64) - axes[a].numpy().astype(np.float64)).max() <= eb_abs


def _block_span(blob, i):
    h = P.parse_header(blob[:46], len(blob))
    tab = np.frombuffer(blob, dtype="<u8", count=h.block_count + 1, offset=46)
    return h.table_end + int(tab[i]), h.table_end + int(tab[i + 1])


def test_streamed_errors_match_one_shot(blob):
    h = P.parse_header(blob[:46], len(blob))
    nb = h.block_count
    cases = []
    # a block's unique count above its particle count, in a late chunk
    b = bytearray(blob)
    s0, _ = _block_span(blob, nb - 3)
    b[s0 + 4: s0 + 8] = (0xFFFF).to_bytes(4, "little")
    cases.append(bytes(b))
    # two bad blocks in different chunks: the first one is reported
    b2 = bytearray(b)
    s1, _ = _block_span(blob, nb // 3)
    b2[s1: s1 + 4] = (5).to_bytes(4, "little")
    cases.append(bytes(b2))
    # a non-finite bound in a middle block
    b3 = bytearray(blob)
    s2, _ = _block_span(blob, nb // 2)
    b3[s2 + 8: s2 + 12] = np.array([np.inf], dtype="<f4").tobytes()
    cases.append(bytes(b3))
    # broken table order (the one-shot path handles it)
    b4 = bytearray(blob)
    o = 46 + 8 * (nb // 2)
    b4[o: o + 8] = (h.payload_len + 1).to_bytes(8, "little")
    cases.append(bytes(b4))
    # a corrupted particle count (high bits of header bytes 30-37): no
    # terabyte-sized pinned buffers, the reference's boundary error
    b5 = bytearray(blob)
    b5[36] ^= 0x40
    cases.append(bytes(b5))
    b6 = bytearray(blob)
    b6[30:38] = (h.particle_count + 5000).to_bytes(8, "little")
    cases.append(bytes(b6))
    for c in cases:
        e_stream = _err(lambda: gz.decompress(c))
        e_dev = _err(lambda: _one_shot(c))
        assert e_stream is not None and e_stream == e_dev, (e_stream, e_dev)


def test_range_decode_any_order_matches_one_shot(blob):
    """gpzb_decompress_range_async (include/gpzb.h): ranges of one container,
    issued in any order on one stream, give the one-shot result and outcome."""
    import ctypes

    from paper_2508_10305_b200 import _lib
    from paper_2508_10305_b200._lib import lib

    cases = [blob]
    b = bytearray(blob)
    h = P.parse_header(blob[:46], len(blob))
    s0, _ = _block_span(blob, h.block_count // 2)
    b[s0: s0 + 4] = (7).to_bytes(4, "little")  # a bad count in a middle block
    cases.append(bytes(b))
    for data in cases:
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
        h = P.parse_header(data[:46], len(data))
        n = h.particle_count
        outs = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(h.dims)]
        wsb = ctypes.c_uint64()
        assert lib.gpzb_decompress_workspace(ctypes.byref(h), ctypes.byref(wsb)) == 0
        ws = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
        stream = torch.cuda.current_stream().cuda_stream
        nb = h.block_count
        cuts = [0, nb // 5, nb // 2, nb - 3, nb]
        ranges = list(zip(cuts[:-1], cuts[1:]))[::-1]  # last range first
        for i, (b0, b1) in enumerate(ranges):
            st = lib.gpzb_decompress_range_async(t.data_ptr(), t.numel(), ctypes.byref(h),
                                                 _lib.ptr_array([o.data_ptr() for o in outs]), n, None,
                                                 ws.data_ptr(), ws.numel(), b0, b1, int(i == 0), stream)
            assert st == 0
        res = _lib.Result()
        lib.gpzb_decompress_result(ws.data_ptr(), ws.numel(), ctypes.byref(h), stream, ctypes.byref(res))
        err = _err(lambda: _one_shot(data))
        if err is None:
            assert res.status == 0
            want = _one_shot(data)
            for a in range(h.dims):
                assert torch.equal(outs[a], want.axes[a])
        else:
            assert res.status != 0
            got = _err(lambda: P._check(res.status, res))
            assert got == err, (got, err)
