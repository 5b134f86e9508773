"""Stage-level entry points on the device, for per-stage parity with the
reference's quantizer / container modules (include/gpzb.h "stage-level
entry points").  The compress path fuses these stages into its own kernels;
these calls run one stage on its own:

* ``block_geometry``  <- quantizer.block_bounds + derive_geometry (quantizer.py:51-129)
* ``quantize``        <- quantizer.quantize_block, codes in input order (quantizer.py:223-247)
* ``encode_payloads`` <- pipeline._encode_block for every block (pipeline.py:38-70)
* ``scan_sizes``      <- container.compact's offsets (container.py:203-208)
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import lib
from .model import Dataset
from .pipeline import _as_dataset, _check, _device_axes, _stream, _workspace

__all__ = ["block_geometry", "quantize", "encode_payloads", "scan_sizes"]


def _prep(ds, block_size: int):
    ds = _as_dataset(ds)
    axes = _device_axes(ds)
    ws_bytes = ctypes.c_uint64()
    _check(lib.gpzb_compress_workspace(ds.count, ds.dims, ds.precision.value, block_size, ctypes.byref(ws_bytes)))
    return ds, axes, _workspace(ws_bytes.value)


def block_geometry(ds: Dataset, eb_abs: float, block_size: int = 1024, target: int = 32) -> dict:
    """Per block and axis: ``lohi`` [B, dims, 2] float64 (the block's exact
    min / max), ``Q`` and ``N`` [B, dims] (bins, segments) and ``log2m``
    [B, dims] — BlockGeometry of every block, as CUDA tensors."""
    ds, axes, ws = _prep(ds, block_size)
    nb = (ds.count + block_size - 1) // block_size
    dev = ws.device
    out = {"lohi": torch.empty(nb, ds.dims, 2, dtype=torch.float64, device=dev),
           "Q": torch.empty(nb, ds.dims, dtype=torch.int64, device=dev),
           "N": torch.empty(nb, ds.dims, dtype=torch.int64, device=dev),
           "log2m": torch.empty(nb, ds.dims, dtype=torch.uint8, device=dev)}
    res = _lib.Result()
    st = lib.gpzb_block_geometry(_lib.ptr_array([a.data_ptr() for a in axes]), ds.dims, ds.precision.value,
                                 ds.count, block_size, target, float(eb_abs), out["lohi"].data_ptr(),
                                 out["Q"].data_ptr(), out["N"].data_ptr(), out["log2m"].data_ptr(), ws.data_ptr(),
                                 ws.numel(), _stream(), ctypes.byref(res))
    _check(st, res)
    return out


def quantize(ds: Dataset, eb_abs: float, block_size: int = 1024, target: int = 32, lohi=None):
    """(seg_ids, offsets) of every particle in input order, as int64 CUDA
    tensors holding the u64 codes.  ``lohi``: carried block bounds (from
    ``block_geometry`` of another dataset), else each block's own."""
    ds, axes, ws = _prep(ds, block_size)
    dev = ws.device
    seg = torch.empty(max(ds.count, 1), dtype=torch.int64, device=dev)
    off = torch.empty(max(ds.count, 1), dtype=torch.int64, device=dev)
    if lohi is not None:
        lohi = lohi.to(device=dev, dtype=torch.float64).contiguous()
    res = _lib.Result()
    st = lib.gpzb_quantize(_lib.ptr_array([a.data_ptr() for a in axes]), ds.dims, ds.precision.value, ds.count,
                           block_size, target, float(eb_abs), lohi.data_ptr() if lohi is not None else None,
                           seg.data_ptr(), off.data_ptr(), ws.data_ptr(), ws.numel(), _stream(), ctypes.byref(res))
    _check(st, res)
    return seg[: ds.count], off[: ds.count]


def encode_payloads(ds: Dataset, eb_abs: float, block_size: int = 1024, target: int = 32,
                    preserve_order: bool = False):
    """Every block's serialised payload (``_encode_block(slice, eb_abs, cfg,
    prec)``) back to back, and the (B + 1) int64 offsets where each starts
    (the last = the total), as CUDA tensors: the container minus its global
    header."""
    ds, axes, ws = _prep(ds, block_size)
    nb = (ds.count + block_size - 1) // block_size
    bound = ctypes.c_uint64()
    _check(lib.gpzb_compress_bound(ds.count, ds.dims, ds.precision.value, block_size, target, int(preserve_order),
                                   ctypes.byref(bound)))
    cap = max(bound.value - 46 - 8 * (nb + 1), 1)
    payloads = torch.empty(cap, dtype=torch.uint8, device=ws.device)
    offsets = torch.empty(nb + 1, dtype=torch.int64, device=ws.device)
    res = _lib.Result()
    st = lib.gpzb_encode_payloads(_lib.ptr_array([a.data_ptr() for a in axes]), ds.dims, ds.precision.value,
                                  ds.count, block_size, target, int(preserve_order), float(eb_abs),
                                  payloads.data_ptr(), cap, offsets.data_ptr(), ws.data_ptr(), ws.numel(), _stream(),
                                  ctypes.byref(res))
    _check(st, res)
    return payloads[: res.out_len].clone(), offsets


def scan_sizes(sizes: torch.Tensor) -> torch.Tensor:
    """offsets[0] = 0, offsets[i + 1] = offsets[i] + sizes[i] (int64 CUDA
    tensors) with the K3a decoupled look-back scan."""
    sizes = sizes.to(dtype=torch.int64).contiguous()
    if not sizes.is_cuda:
        sizes = sizes.cuda()
    nb = sizes.numel()
    out = torch.empty(nb + 1, dtype=torch.int64, device=sizes.device)
    wsb = ctypes.c_uint64()
    _check(lib.gpzb_scan_workspace(nb, ctypes.byref(wsb)))
    ws = _workspace(wsb.value, slot=99)
    _check(lib.gpzb_scan_sizes(sizes.data_ptr(), nb, out.data_ptr(), ws.data_ptr(), ws.numel(), _stream()))
    return out
