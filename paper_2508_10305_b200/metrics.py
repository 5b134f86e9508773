"""Rate-distortion evaluation and error-bound verification on the GPU.

Mirrors the reference's ``gpz.metrics`` (metrics.py:1-200): same names,
signatures, dataclasses, CSV format and error classes.  The per-particle
work — block pairing (quantize both datasets with the original block's
geometry, order each by (seg_id, offset, index)), squared-error sums, field
ranges, the maximum error and the list of bound violations — runs in the
K5 kernels of ``_gpzb.so`` (gpzb_pair_blocks / gpzb_pair_stats); this module
moves buffers and does the scalar arithmetic of the final formulas.

Inputs may be numpy arrays or torch tensors (host or CUDA); pairings come
back as numpy int64 arrays like the reference's, or as CUDA tensors from
``pair_blocks_device``.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import lib
from .errors import DomainError
from .model import CompressConfig, Dataset, EbMode, Precision
from .pipeline import _check, _device, _stream, resolve_absolute_bound

__all__ = [
    "compression_ratio",
    "bitrate",
    "pair_blocks",
    "pair_blocks_device",
    "nrmse",
    "aggregate_psnr",
    "verify_bound",
    "BoundReport",
    "RateDistortionRow",
    "evaluate",
    "CSV_HEADER",
]


def compression_ratio(original_bytes: int, compressed_bytes: int) -> float:
    """metrics.compression_ratio (metrics.py:36-39)."""
    if compressed_bytes == 0:
        raise DomainError("compressed size of zero bytes")
    return original_bytes / compressed_bytes


def bitrate(compressed_bytes: int, particle_count: int) -> float:
    """Average compressed bits per particle (metrics.py:42-46)."""
    if particle_count == 0:
        raise DomainError("bitrate of zero particles")
    return 8.0 * compressed_bytes / particle_count


def _dev_array(a, dtype=None) -> torch.Tensor:
    dev = _device()
    if isinstance(a, torch.Tensor):
        t = a.to(dev, non_blocking=True) if (not a.is_cuda or a.device != dev) else a
    else:
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def _prec_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.F32
    if t.dtype == torch.float64:
        return _lib.F64
    raise DomainError(f"unsupported coordinate dtype {t.dtype}")


_PWS: dict = {}


def _pair_ws(count: int, dims: int) -> torch.Tensor:
    need = ctypes.c_uint64()
    _check(lib.gpzb_pair_workspace(max(count, 1), dims, ctypes.byref(need)))
    dev = _device()
    buf = _PWS.get(dev.index)
    if buf is None or buf.numel() < need.value:
        buf = torch.empty(max(need.value, 1 << 16), dtype=torch.uint8, device=dev)
        _PWS[dev.index] = buf
    return buf


def pair_blocks_device(original: Dataset, reconstructed: Dataset, cfg: CompressConfig,
                       eb_abs: float | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """pair_blocks with the index arrays left on the device (int64 CUDA tensors)."""
    if original.count != reconstructed.count or original.dims != reconstructed.dims:
        raise DomainError("datasets differ in shape, cannot pair")
    if eb_abs is None:
        eb_abs = resolve_absolute_bound(original, cfg)
    orig = [_dev_array(a) for a in original.axes]
    rec = [_dev_array(a) for a in reconstructed.axes]
    n = original.count
    oi = torch.empty(n, dtype=torch.int64, device=_device())
    ri = torch.empty(n, dtype=torch.int64, device=_device())
    if n == 0:
        return oi, ri
    ws = _pair_ws(n, original.dims)
    res = _lib.Result()
    st = lib.gpzb_pair_blocks(_lib.ptr_array([a.data_ptr() for a in orig]),
                              _lib.ptr_array([a.data_ptr() for a in rec]), original.dims,
                              original.precision.value, _prec_code(rec[0]), n, float(eb_abs), cfg.block_size,
                              cfg.target_segs_per_axis, oi.data_ptr(), ri.data_ptr(), ws.data_ptr(), ws.numel(),
                              _stream(), ctypes.byref(res))
    if st == _lib.WIDTH and res.block >= 0:  # derive_geometry raises without a block prefix (metrics.py:76-78)
        res.block = -1
    _check(st, res)
    return oi, ri


def pair_blocks(original: Dataset, reconstructed: Dataset, cfg: CompressConfig,
                eb_abs: float | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Index arrays pairing original and reconstructed particles (metrics.py:54-81).

    Both datasets must share block boundaries; each block is quantized with
    the original's bounds so equal values land on equal codes.
    """
    oi, ri = pair_blocks_device(original, reconstructed, cfg, eb_abs)
    return oi.cpu().numpy(), ri.cpu().numpy()


def _index_array(idx, size: int) -> torch.Tensor:
    """A pairing index vector on the device with numpy's fancy-indexing rules
    (metrics.py:93-94): negative indices count from the end, anything outside
    [-size, size) raises IndexError."""
    t = _dev_array(idx, torch.int64)
    if t.numel():
        lo, hi = int(t.min()), int(t.max())
        if lo < -size or hi >= size:
            bad = lo if lo < -size else hi
            raise IndexError(f"index {bad} is out of bounds for axis 0 with size {size}")
        if lo < 0:
            t = torch.where(t < 0, t + size, t)
    return t


def _stats(orig: list, rec: list, pairing, eb_abs: float, want_violations: bool):
    """K5b over paired values: (stats vector, violations array [k, 3] or None)."""
    dims = len(orig)
    n_o, n_r = int(orig[0].numel()), int(rec[0].numel())
    oi = ri = None
    if pairing is None:
        # elementwise o - r: numpy broadcasting rejects unequal lengths (metrics.py:90-97)
        if n_o != n_r:
            raise ValueError(f"operands could not be broadcast together with shapes ({n_o},) ({n_r},)")
        n = n_o
    else:
        oi = _index_array(pairing[0], n_o)
        ri = _index_array(pairing[1], n_r)
        if oi.numel() != ri.numel():
            raise ValueError(f"operands could not be broadcast together with shapes ({oi.numel()},) ({ri.numel()},)")
        n = int(oi.numel())
    ws = _pair_ws(n, dims)
    stats = (ctypes.c_double * (1 + 3 * dims))()
    count = ctypes.c_uint64()
    cap = 4096 if want_violations else 0
    while True:
        viol = torch.empty(max(3 * cap, 3), dtype=torch.int64, device=_device())
        st = lib.gpzb_pair_stats(_lib.ptr_array([a.data_ptr() for a in orig]),
                                 _lib.ptr_array([a.data_ptr() for a in rec]), dims, _prec_code(orig[0]),
                                 _prec_code(rec[0]), n, oi.data_ptr() if oi is not None else None,
                                 ri.data_ptr() if ri is not None else None, float(eb_abs),
                                 viol.data_ptr() if cap else None, cap, ws.data_ptr(), ws.numel(), _stream(),
                                 stats, ctypes.byref(count))
        _check(st)
        if not want_violations or count.value <= cap:
            break
        cap = int(count.value)
    v = None
    if want_violations:
        v = viol[: 3 * count.value].view(-1, 3).cpu().numpy() if count.value else np.zeros((0, 3), np.int64)
    return list(stats), v


def nrmse(field_original, field_reconstructed, pairing=None) -> float:
    """Root-mean-square error normalized by the original field's range (metrics.py:84-104).

    Σ (o - r)^2 and the range come from K5b in float64; the summation order
    differs from numpy's pairwise sum, so the result agrees to ~1e-12 relative.
    """
    o = _dev_array(field_original)
    r = _dev_array(field_reconstructed)
    if o.dtype not in (torch.float32, torch.float64):
        o = o.to(torch.float64)
    if r.dtype not in (torch.float32, torch.float64):
        r = r.to(torch.float64)
    n = o.numel() if pairing is None else int(len(pairing[0]))
    if n == 0:
        return 0.0
    st, _ = _stats([o], [r], pairing, math.inf, False)
    rmse = math.sqrt(st[1] / n)
    span = st[3] - st[2]
    if span <= 0.0:
        if rmse == 0.0:
            return 0.0
        raise DomainError("degenerate field range with nonzero error")
    return rmse / span


def aggregate_psnr(nrmse_values) -> float:
    """-20 log10 of the root mean square of the per-field NRMSE values (metrics.py:107-119).

    Returns +inf when every NRMSE is zero (distortion-free fields).
    """
    values = [float(v) for v in nrmse_values]
    if not values:
        raise DomainError("aggregate PSNR of no fields")
    mean_sq = sum(v * v for v in values) / len(values)
    if mean_sq == 0.0:
        return math.inf
    return -20.0 * math.log10(math.sqrt(mean_sq))


@dataclass(frozen=True)
class BoundReport:
    max_err: float
    violations: list  # (axis, original index, |error|)
    checked: int

    @property
    def ok(self) -> bool:
        return not self.violations


def _pair_and_stats(original: Dataset, reconstructed: Dataset, eb_abs: float, cfg: CompressConfig,
                    want_violations: bool):
    oi, ri = pair_blocks_device(original, reconstructed, cfg, eb_abs)
    orig = [_dev_array(a) for a in original.axes]
    rec = [_dev_array(a) for a in reconstructed.axes]
    return _stats(orig, rec, (oi, ri), eb_abs, want_violations)


def _report(stats, viol, eb_abs, original: Dataset) -> BoundReport:
    # the reference lists violations axis by axis in pairing order (metrics.py:140-151)
    order = np.lexsort((viol[:, 0] & ((1 << 56) - 1), viol[:, 0] >> 56)) if len(viol) else []
    violations = [(int(viol[i, 0] >> 56), int(viol[i, 1]), float(np.int64(viol[i, 2]).view(np.float64)))
                  for i in order]
    max_err = stats[0] if original.count else 0.0
    return BoundReport(max_err=float(max_err), violations=violations, checked=original.count * original.dims)


def verify_bound(original: Dataset, reconstructed: Dataset, eb_abs: float, cfg: CompressConfig) -> BoundReport:
    """Check |p' - p| <= eb_abs per axis under block-multiset pairing (metrics.py:131-152)."""
    if original.count == 0:
        return BoundReport(max_err=0.0, violations=[], checked=0)
    stats, viol = _pair_and_stats(original, reconstructed, eb_abs, cfg, True)
    return _report(stats, viol, eb_abs, original)


CSV_HEADER = "eb,eb_abs,cr,bitrate,nrmse,psnr,max_err"


@dataclass(frozen=True)
class RateDistortionRow:
    eb: float
    eb_abs: float
    cr: float
    bitrate: float
    nrmse_per_axis: tuple
    psnr: float
    max_err: float

    def to_csv(self) -> str:
        nrmse_field = ";".join(f"{v:.6e}" for v in self.nrmse_per_axis)
        psnr = "inf" if math.isinf(self.psnr) else f"{self.psnr:.4f}"
        return (
            f"{self.eb:g},{self.eb_abs:.12e},{self.cr:.4f},{self.bitrate:.4f},"
            f"{nrmse_field},{psnr},{self.max_err:.6e}"
        )


def evaluate(original: Dataset, reconstructed: Dataset, compressed_bytes: int, eb: float, eb_abs: float,
             cfg: CompressConfig) -> RateDistortionRow:
    """One rate-distortion table row for a (dataset, bound) pair (metrics.py:175-200).

    One pairing pass serves both the NRMSE per axis and the bound check.
    """
    if original.count == 0:
        per_axis = tuple(0.0 for _ in range(original.dims))
        max_err = 0.0
    else:
        stats, _ = _pair_and_stats(original, reconstructed, eb_abs, cfg, False)
        per_axis = []
        for a in range(original.dims):
            sq, lo, hi = stats[1 + 3 * a], stats[2 + 3 * a], stats[3 + 3 * a]
            rmse = math.sqrt(sq / original.count)
            span = hi - lo
            if span <= 0.0:
                if rmse != 0.0:
                    raise DomainError("degenerate field range with nonzero error")
                per_axis.append(0.0)
            else:
                per_axis.append(rmse / span)
        per_axis = tuple(per_axis)
        max_err = stats[0]
    return RateDistortionRow(
        eb=eb,
        eb_abs=eb_abs,
        cr=compression_ratio(original.nbytes, compressed_bytes),
        bitrate=bitrate(compressed_bytes, original.count),
        nrmse_per_axis=per_axis,
        psnr=aggregate_psnr(per_axis),
        max_err=float(max_err),
    )
