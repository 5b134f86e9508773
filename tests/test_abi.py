"""C-ABI library and host-logic checks that need no GPU."""

import ctypes
import os
import re
import struct

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    import paper_2508_10305_b200._lib as L

    header = open(os.path.join(ROOT, "include", "gpzb.h")).read()
    declared = set(re.findall(r"\b(gpzb_\w+)\s*\(", header))
    assert len(declared) >= 14
    so = ctypes.CDLL(L.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(so, name), name
    assert set(L.SIGNATURES) == declared


def test_library_is_sm100a():
    import subprocess

    import paper_2508_10305_b200._lib as L

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _hdr(**kw):
    f = dict(magic=b"GPZ1", ver=1, dims=3, prec=0, flags=0, mode=1, eb=1e-3, eb_abs=1.25e-3, bs=1024, n=10, b=1)
    f.update(kw)
    return struct.pack("<4sHBBBBddIQQ", f["magic"], f["ver"], f["dims"], f["prec"], f["flags"], f["mode"],
                       f["eb"], f["eb_abs"], f["bs"], f["n"], f["b"])


@pytest.mark.parametrize("kw,total,ok", [
    ({}, 46 + 16, True),
    ({"magic": b"GPZ2"}, 62, False),
    ({"ver": 2}, 62, False),
    ({"dims": 4}, 62, False),
    ({"dims": 0}, 62, False),
    ({"prec": 2}, 62, False),
    ({"mode": 2}, 62, False),
    ({"eb_abs": 0.0}, 62, False),
    ({"eb_abs": float("inf")}, 62, False),
    ({"flags": 2}, 62, False),
    ({"b": 5}, 62, False),      # table does not fit
    ({}, 30, False),            # shorter than the global header
])
def test_parse_header_matches_oracle(kw, total, ok):
    from oracle import gpz_oracle as O
    import paper_2508_10305_b200 as gz
    from paper_2508_10305_b200.pipeline import parse_header

    raw = _hdr(**kw)
    data = (raw + bytes(16))[:total] if total >= 46 else raw[:total]
    if ok:
        h = parse_header(data, len(data))
        assert (h.dims, h.block_count, h.table_end) == (3, 1, 62)
    else:
        with pytest.raises(gz.CorruptData):
            parse_header(data, len(data))
        # the oracle raises the same class for the same header (container.py:245-281)
        try:
            O.read_container(data)
        except O.CorruptData:
            pass


def test_compress_bound_covers_worst_case():
    import paper_2508_10305_b200._lib as L

    b = ctypes.c_uint64()
    assert L.lib.gpzb_compress_bound(1024, 3, 0, 1024, 32, 0, ctypes.byref(b)) == 0
    # 46 + 2 table entries + header + 64-bit deltas/offsets + 11-bit counts
    assert b.value >= 46 + 16 + 50 + 8192 + 1408 + 8192
    assert L.lib.gpzb_compress_bound(10, 3, 0, 2048, 32, 0, ctypes.byref(b)) == 0  # K2b / K4b
    assert L.lib.gpzb_compress_bound(10, 3, 0, 1 << 25, 32, 0, ctypes.byref(b)) == L.UNSUPPORTED
    assert L.lib.gpzb_compress_bound(10, 3, 0, 100, 32, 0, ctypes.byref(b)) == L.INVALID


def test_config_validation_mirrors_reference():
    import paper_2508_10305_b200 as gz

    for bad in (dict(error_bound=0.0), dict(error_bound=float("nan")), dict(error_bound=1e-3, block_size=33),
                dict(error_bound=1e-3, target_segs_per_axis=3)):
        with pytest.raises(gz.DomainError):
            gz.CompressConfig(**bad)
    with pytest.raises(gz.DomainError):
        gz.Dataset.from_axes([np.zeros(3), np.zeros(4)])
    with pytest.raises(gz.DomainError):
        gz.Dataset.from_axes([np.zeros(3)] * 4)
    with pytest.raises(gz.DomainError):
        gz.Dataset.from_axes([np.zeros(3, np.int32)])
    assert [(s.start, s.stop) for s in gz.iter_block_slices(10, 4)] == [(0, 4), (4, 8), (8, 10)]


def test_no_cpu_fallback_without_gpu():
    import torch

    import paper_2508_10305_b200 as gz

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="CUDA"):
        gz.compress(gz.Dataset.from_axes([np.zeros(8, np.float32)]), gz.CompressConfig(1e-3))
