"""CPU oracle for the GPZ compress / decompress path — TEST INFRASTRUCTURE ONLY.

This module is the checker the CUDA path is compared against.  Only
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it; the product
package (``paper_2508_10305_b200``) never does, and fails loudly when its
CUDA library is missing instead of routing here.

It restates, in numpy, the algorithm of the reference package ``gpz``
(``/root/reference/pkg/src/gpz``; every function cites the file:line it
follows).  The reference is pure Python + numpy, so "the reference
algorithm" is exactly its float64 arithmetic and its byte format:

* stage 1 quantize  — ``quantizer.py:51-191`` (bounds, guard margin, geometry,
  float64 floor-divide quantization with the edge-snap rule, linearization)
* stage 2 sort      — ``blocksort.py:17-28`` (stable lexicographic (seg, off))
* stage 3 encode    — ``codec.py:53-151`` (RLE, delta, width, LSB-first pack)
* stage 4 compact   — ``container.py:102-303`` (block header, prefix-sum
  offset table, 46-byte global header)
* orchestration     — ``pipeline.py:38-215``
* evaluation        — ``metrics.py:49-152`` (block pairing, NRMSE, PSNR,
  bound check: the checker for the GPU K5 kernels)

Parity is PINNED: ``tests/golden/`` holds containers, reconstructions and
error outcomes produced by the reference itself (``tests/golden/make_golden.py``
imports ``/root/reference/pkg/src/gpz`` in the build container); the
``-m "not gpu"`` suite checks this oracle against every one of them.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np

# --------------------------------------------------------------------------
# error classes (names mirror gpz.errors, errors.py:4-17)


class OracleError(Exception):
    """Base of the oracle's error classes (gpz.errors.GpzError)."""


class DomainError(OracleError):
    pass


class WidthOverflow(OracleError):
    pass


class CorruptData(OracleError):
    pass


# --------------------------------------------------------------------------
# enum codes (model.py:29-53) — these bytes are part of the file format

F32, F64 = 0, 1
ABSOLUTE, RANGE_RELATIVE = 0, 1

_ITEM = {F32: 4, F64: 8}
_NPTYPE = {F32: np.float32, F64: np.float64}
# relative guard per output precision (quantizer.py:41-46)
_GUARD = {F32: 2.0 ** -24 + 2.0 ** -48, F64: 2.0 ** -48}
_TWO64 = 1 << 64

GLOBAL_FMT = "<4sHBBBBddIQQ"          # container.py:57
GLOBAL_SIZE = struct.calcsize(GLOBAL_FMT)  # 46 bytes
MAGIC = b"GPZ1"
VERSION = 1


@dataclass(frozen=True)
class Config:
    """Mirror of gpz.CompressConfig (model.py:102-123)."""

    error_bound: float
    eb_mode: int = RANGE_RELATIVE
    block_size: int = 1024
    target_segs_per_axis: int = 32
    preserve_order: bool = False

    def __post_init__(self):
        if not (self.error_bound > 0 and math.isfinite(self.error_bound)):
            raise DomainError(f"error_bound must be a positive finite real, got {self.error_bound}")
        if self.block_size <= 0 or self.block_size % 32:
            raise DomainError(f"block_size must be a positive multiple of 32, got {self.block_size}")
        t = self.target_segs_per_axis
        if t < 1 or (t & (t - 1)):
            raise DomainError(f"target_segs_per_axis must be a power of two >= 1, got {t}")


def precision_of(arr) -> int:
    """model.py:41-48"""
    dt = np.dtype(arr.dtype)
    if dt == np.float32:
        return F32
    if dt == np.float64:
        return F64
    raise DomainError(f"unsupported coordinate dtype {dt}")


def check_axes(axes) -> tuple[list[np.ndarray], int]:
    """Dataset invariants (model.py:67-78): 1..3 equal-length finite axes."""
    if not 1 <= len(axes) <= 3:
        raise DomainError(f"dims must be 1, 2 or 3, got {len(axes)}")
    prec = precision_of(np.asarray(axes[0]))
    arrs = [np.ascontiguousarray(a, dtype=_NPTYPE[prec]) for a in axes]
    if len({a.shape for a in arrs}) != 1 or arrs[0].ndim != 1:
        raise DomainError("all axes must be 1-D arrays of identical length")
    for i, a in enumerate(arrs):
        if a.size and not np.isfinite(a).all():
            raise DomainError(f"axis {i} contains non-finite coordinates")
    return arrs, prec


# --------------------------------------------------------------------------
# stage 1 — bounds, geometry, quantization


def absolute_bound(axes, cfg: Config) -> float:
    """model.py:183-199 (joint range over all axes in REL mode)."""
    if cfg.eb_mode == ABSOLUTE:
        return float(cfg.error_bound)
    if axes[0].size == 0:
        raise DomainError("range-relative bound is undefined for an empty dataset")
    lo = min(float(a.min()) for a in axes)
    hi = max(float(a.max()) for a in axes)
    span = hi - lo
    return float(cfg.error_bound) * (span if span > 0.0 else 1.0)


def inner_bound(eb_abs: float, lo: float, hi: float, prec: int) -> float:
    """effective_bound, quantizer.py:60-68: eb minus the guard margin."""
    scale = max(abs(lo), abs(hi)) + 2.0 * eb_abs
    margin = scale * _GUARD[prec]
    return 0.5 * eb_abs if margin >= 0.5 * eb_abs else eb_abs - margin


def bin_count(lo: float, hi: float, eb_abs: float, prec: int) -> int:
    """axis_bin_count, quantizer.py:71-86."""
    span = hi - lo
    if span <= 0.0:
        return 1
    ratio = span / (2.0 * inner_bound(eb_abs, lo, hi, prec))
    if not ratio < 18446744073709551616.0:
        raise WidthOverflow(f"axis range {span:g} over bound {eb_abs:g} exceeds 64-bit bin indices")
    return int(math.floor(ratio)) + 1


@dataclass(frozen=True)
class Geometry:
    """BlockGeometry (model.py:126-162) reduced to what the codec needs."""

    mins: tuple
    maxs: tuple
    Q: tuple      # bins per axis
    m: tuple      # power-of-two segment sizes
    N: tuple      # segment counts

    @property
    def bits(self):
        return tuple(x.bit_length() - 1 for x in self.m)

    @property
    def n_segments(self):
        return math.prod(self.N)

    @property
    def n_offsets(self):
        return math.prod(self.m)


def geometry(mins, maxs, eb_abs: float, target: int, prec: int) -> Geometry:
    """derive_geometry, quantizer.py:89-129."""
    if not eb_abs > 0:
        raise DomainError(f"absolute bound must be positive, got {eb_abs}")
    Qs, ms, Ns = [], [], []
    for lo, hi in zip(mins, maxs):
        q = bin_count(lo, hi, eb_abs, prec)
        per = -(-q // target)
        m = 1 << (per - 1).bit_length()
        Qs.append(q)
        ms.append(m)
        Ns.append(-(-q // m))
    g = Geometry(tuple(mins), tuple(maxs), tuple(Qs), tuple(ms), tuple(Ns))
    if g.n_segments > _TWO64 or g.n_offsets > _TWO64:
        raise WidthOverflow(
            f"geometry needs {g.n_segments} segments x {g.n_offsets} offsets, "
            "beyond the 64-bit linearization range")
    return g


def _midpoints(q: np.ndarray, lo: float, eb_int: float, prec: int) -> np.ndarray:
    """_axis_reconstruction, quantizer.py:132-139 (what the decoder emits)."""
    v = lo + (q.astype(np.float64) + 0.5) * (2.0 * eb_int)
    return v.astype(np.float32).astype(np.float64) if prec == F32 else v


def quantize_axis(vals: np.ndarray, lo: float, hi: float, Q: int, eb_abs: float, prec: int) -> np.ndarray:
    """_quantize_axis, quantizer.py:142-173: float64 floor-divide + edge snap."""
    x = np.asarray(vals, dtype=np.float64)
    eb_int = inner_bound(eb_abs, lo, hi, prec)
    qf = np.floor((x - lo) / (2.0 * eb_int))
    qf = np.minimum(np.maximum(qf, 0.0), float(Q - 1))
    q = qf.astype(np.uint64)
    rec = _midpoints(q, lo, eb_int, prec)
    err = np.abs(rec - x)
    over = np.nonzero(err > eb_abs)[0]
    if over.size and Q <= (1 << 62):
        step = np.where(rec[over] > x[over], -1, 1)
        cand = np.clip(q[over].astype(np.int64) + step, 0, Q - 1).astype(np.uint64)
        cerr = np.abs(_midpoints(cand, lo, eb_int, prec) - x[over])
        take = cerr < err[over]
        q[over[take]] = cand[take]
    return q


def linearize(qs, g: Geometry):
    """_split_and_linearize, quantizer.py:176-191."""
    seg = np.zeros(qs[0].shape, np.uint64)
    off = np.zeros(qs[0].shape, np.uint64)
    stride, shift = 1, 0
    for a, q in enumerate(qs):
        b = g.bits[a]
        seg += (q >> np.uint64(b)) * np.uint64(stride)
        off |= (q & np.uint64(g.m[a] - 1)) << np.uint64(shift)
        stride *= g.N[a]
        shift += b
    return seg, off


def split_codes(seg: np.ndarray, off: np.ndarray, g: Geometry):
    """_delinearize, quantizer.py:194-213: per-axis bin indices."""
    rest = seg.astype(np.uint64).copy()
    off = off.astype(np.uint64)
    out, shift = [], 0
    for a in range(len(g.N)):
        if a + 1 < len(g.N):
            s = rest % np.uint64(g.N[a])
            rest //= np.uint64(g.N[a])
        else:
            s = rest
        b = g.bits[a]
        o = (off >> np.uint64(shift)) & np.uint64(g.m[a] - 1)
        out.append((s << np.uint64(b)) | o)
        shift += b
    return out


# --------------------------------------------------------------------------
# stage 3 — integer codecs


def bit_width(v: np.ndarray) -> int:
    """width_for, codec.py:107-112."""
    return int(np.max(v)).bit_length() if v.size else 0


def pack(v: np.ndarray, w: int) -> bytes:
    """pack_fixed, codec.py:115-129: LSB-first, back to back, zero pad.

    Builds the bit string from each value's little-endian byte image.
    """
    v = np.ascontiguousarray(v, dtype=np.uint64)
    if not 0 <= w <= 64:
        raise DomainError(f"bit width must be in 0..64, got {w}")
    if w == 0:
        if v.size and int(v.max()) != 0:
            raise DomainError("nonzero value in a zero-width stream")
        return b""
    if w < 64 and v.size and int(v.max()) >> w:
        raise DomainError(f"value exceeds {w} bits")
    allbits = np.unpackbits(v.astype("<u8").view(np.uint8).reshape(-1, 8), axis=1, bitorder="little")
    return np.packbits(allbits[:, :w].reshape(-1), bitorder="little").tobytes()


def unpack(raw: bytes, n: int, w: int) -> np.ndarray:
    """unpack_fixed, codec.py:132-151 (dirty padding is corruption)."""
    if not 0 <= w <= 64:
        raise CorruptData(f"bit width must be in 0..64, got {w}")
    if w == 0 or n == 0:
        if len(raw):
            raise CorruptData("zero-width or empty stream carries payload bytes")
        return np.zeros(n, np.uint64)
    if len(raw) != (n * w + 7) // 8:
        raise CorruptData(f"packed stream is {len(raw)} bytes, expected {(n * w + 7) // 8}")
    bits = np.unpackbits(np.frombuffer(raw, np.uint8), bitorder="little")
    if bits[n * w:].any():
        raise CorruptData("nonzero padding bits in packed stream")
    full = np.zeros((n, 64), np.uint8)
    full[:, :w] = bits[: n * w].reshape(n, w)
    return np.packbits(full, axis=1, bitorder="little").view("<u8").reshape(n).astype(np.uint64)


def runs(sorted_ids: np.ndarray):
    """rle_encode, codec.py:53-79: unique ids and run lengths."""
    n = sorted_ids.size
    if n == 0:
        return sorted_ids[:0].copy(), np.zeros(0, np.int64)
    if np.any(sorted_ids[1:] < sorted_ids[:-1]):
        raise DomainError("run-length input must be nondecreasing (sort stage defect)")
    head = np.ones(n, bool)
    head[1:] = sorted_ids[1:] != sorted_ids[:-1]
    starts = np.nonzero(head)[0]
    return sorted_ids[starts], np.diff(np.append(starts, n))


# --------------------------------------------------------------------------
# stage 4 — block payloads and the container


def block_header_fmt(dims: int, prec: int, preserve: bool) -> str:
    """_header_fmt, container.py:62-67."""
    axis = "ffBI" if prec == F32 else "ddBI"
    return "<II" + axis * dims + ("BBBB" if preserve else "BBB")


def encode_block(block_axes, eb_abs: float, cfg: Config, prec: int) -> bytes:
    """_encode_block, pipeline.py:38-70 — all four stages for one block."""
    if not block_axes or block_axes[0].size == 0:
        raise DomainError("block bounds of an empty block are undefined")
    mins = tuple(float(a.min()) for a in block_axes)       # quantizer.py:51-57
    maxs = tuple(float(a.max()) for a in block_axes)
    g = geometry(mins, maxs, eb_abs, cfg.target_segs_per_axis, prec)
    for i, a in enumerate(block_axes):                     # quantizer.py:230-232
        if not np.isfinite(a).all():
            raise DomainError(f"axis {i} contains non-finite coordinates")
    qs = [quantize_axis(a, g.mins[i], g.maxs[i], g.Q[i], eb_abs, prec) for i, a in enumerate(block_axes)]
    seg, off = linearize(qs, g)
    n = seg.size
    order = np.lexsort((off, seg)) if n > 1 else np.arange(n)  # blocksort.py:17-28
    seg, off = seg[order], off[order]
    uniq, counts = runs(seg)
    deltas = uniq.copy()
    if deltas.size > 1:
        deltas[1:] = uniq[1:] - uniq[:-1]                  # codec.py:93-100
    streams = [(deltas, bit_width(deltas)), (counts.astype(np.uint64), bit_width(counts)),
               (off, bit_width(off))]
    if cfg.preserve_order:
        ranks = order.astype(np.uint64)                    # quantizer.py:240-241
        streams.append((ranks, bit_width(ranks)))
    fields = [n, int(uniq.size)]
    for a in range(len(block_axes)):
        fields += [g.mins[a], g.maxs[a], g.bits[a], g.N[a]]
    fields += [w for _, w in streams]
    head = struct.pack(block_header_fmt(len(block_axes), prec, cfg.preserve_order), *fields)
    return head + b"".join(pack(v, w) for v, w in streams)


def compress(axes, cfg: Config) -> bytes:
    """pipeline.compress, pipeline.py:73-103 (serial: output is worker-independent)."""
    axes, prec = check_axes(axes)
    count = axes[0].size
    eb_abs = absolute_bound(axes, cfg) if count else float(cfg.error_bound)
    payloads = []
    for i, start in enumerate(range(0, count, cfg.block_size)):
        sl = slice(start, min(start + cfg.block_size, count))
        try:
            payloads.append(encode_block([a[sl] for a in axes], eb_abs, cfg, prec))
        except (DomainError, WidthOverflow) as exc:
            raise type(exc)(f"block {i}: {exc}") from None
    return assemble(len(axes), prec, cfg, eb_abs, count, payloads)


def assemble(dims, prec, cfg: Config, eb_abs, count, payloads) -> bytes:
    """compact + write_container, container.py:203-230."""
    table = np.zeros(len(payloads) + 1, "<u8")
    np.cumsum([len(p) for p in payloads], out=table[1:])
    head = struct.pack(GLOBAL_FMT, MAGIC, VERSION, dims, prec, 1 if cfg.preserve_order else 0,
                       cfg.eb_mode, float(cfg.error_bound), eb_abs, cfg.block_size, count, len(payloads))
    return head + table.tobytes() + b"".join(payloads)


@dataclass(frozen=True)
class Header:
    dims: int
    prec: int
    preserve: bool
    eb_mode: int
    eb: float
    eb_abs: float
    block_size: int
    count: int
    blocks: int


def read_container(data: bytes):
    """read_container, container.py:245-303: header, table, payload."""
    if len(data) < GLOBAL_SIZE:
        raise CorruptData(f"container of {len(data)} bytes, global header needs {GLOBAL_SIZE}")
    magic, ver, dims, prec, flags, mode, eb, eb_abs, bs, count, nblk = struct.unpack_from(GLOBAL_FMT, data)
    if magic != MAGIC:
        raise CorruptData(f"bad magic {magic!r} at byte 0")
    if ver != VERSION:
        raise CorruptData(f"unsupported container version {ver}")
    if not 1 <= dims <= 3:
        raise CorruptData(f"dims {dims} outside 1..3")
    if prec not in (F32, F64) or mode not in (ABSOLUTE, RANGE_RELATIVE):
        raise CorruptData(f"bad precision/eb_mode code {prec}/{mode}")
    if not (math.isfinite(eb_abs) and eb_abs > 0):
        raise CorruptData(f"absolute bound {eb_abs} is not a positive real")
    if flags & ~1:
        raise CorruptData(f"unknown flag bits 0x{flags:02x}")
    table_end = GLOBAL_SIZE + (nblk + 1) * 8
    if len(data) < table_end:
        raise CorruptData(f"container truncated inside the offset table at byte {len(data)}")
    table = np.frombuffer(data, "<u8", count=nblk + 1, offset=GLOBAL_SIZE)
    if table[0] != 0:
        raise CorruptData("offset table must start at 0")
    if np.any(table[1:] < table[:-1]):
        raise CorruptData("offset table is not nondecreasing")
    payload = data[table_end:]
    if int(table[-1]) != len(payload):
        raise CorruptData(f"offset table ends at {int(table[-1])} but payload holds {len(payload)} bytes")
    h = Header(dims, prec, bool(flags & 1), mode, eb, eb_abs, bs, count, nblk)
    return h, table, payload


def decode_block(p: bytes, h: Header) -> list[np.ndarray]:
    """_decode_block, pipeline.py:106-157 with parse_block (container.py:128-200)."""
    fmt = block_header_fmt(h.dims, h.prec, h.preserve)
    hsz = struct.calcsize(fmt)
    if len(p) < hsz:
        raise CorruptData(f"block payload of {len(p)} bytes, header needs {hsz}")
    f = struct.unpack_from(fmt, p)
    n, U = f[0], f[1]
    mins = [float(f[2 + 4 * a]) for a in range(h.dims)]
    maxs = [float(f[3 + 4 * a]) for a in range(h.dims)]
    bits = [int(f[4 + 4 * a]) for a in range(h.dims)]
    Ns = [int(f[5 + 4 * a]) for a in range(h.dims)]
    widths = list(f[2 + 4 * h.dims:])
    if U > n:
        raise CorruptData(f"{U} unique ids for {n} particles")
    if any(w > 64 for w in widths):
        raise CorruptData("stream width exceeds 64 bits")
    for a in range(h.dims):
        if Ns[a] < 1 and n > 0:
            raise CorruptData(f"axis {a} has no segments")
        if bits[a] > 63:
            raise CorruptData(f"axis {a} offset width {bits[a]} exceeds 63 bits")
        if not (math.isfinite(mins[a]) and math.isfinite(maxs[a]) and mins[a] <= maxs[a]):
            raise CorruptData(f"axis {a} bounds [{mins[a]}, {maxs[a]}] are invalid")
    counts_n = [U, U, n] + ([n] if h.preserve else [])
    cur, raw = hsz, []
    for cnt, w in zip(counts_n, widths):
        nb = (cnt * w + 7) // 8
        chunk = p[cur:cur + nb]
        if len(chunk) != nb:
            raise CorruptData(f"block truncated at byte {cur}")
        raw.append(chunk)
        cur += nb
    if cur != len(p):
        raise CorruptData(f"{len(p) - cur} trailing bytes after block streams")
    deltas = unpack(raw[0], U, widths[0])
    counts = unpack(raw[1], U, widths[1])
    offs = unpack(raw[2], n, widths[2])
    uniq = np.cumsum(deltas, dtype=np.uint64)
    if uniq.size and np.any(uniq[1:] <= uniq[:-1]):
        raise CorruptData("decoded unique ids are not strictly increasing")
    if counts.size and int(counts.min()) < 1:
        raise CorruptData("decoded run length of zero")
    if int(counts.sum(dtype=np.uint64)) != n:
        raise CorruptData(f"run lengths do not cover {n} particles")
    if counts.size and int(counts.max()) >= 1 << 63:
        raise CorruptData("run length beyond any block size")
    seg = np.repeat(uniq, counts.astype(np.int64))
    ms = [1 << b for b in bits]
    Qs = []
    for a in range(h.dims):
        try:
            q = bin_count(mins[a], maxs[a], h.eb_abs, h.prec)
        except OracleError as exc:
            raise CorruptData(str(exc)) from None
        if n and -(-q // ms[a]) != Ns[a]:
            raise CorruptData(f"axis {a}: {Ns[a]} segments inconsistent with {q} bins of size {ms[a]}")
        Qs.append(q)
    g = Geometry(tuple(mins), tuple(maxs), tuple(Qs), tuple(ms), tuple(Ns))
    if n:
        if int(seg.max()) >= g.n_segments:
            raise CorruptData("segment id outside the block geometry")
        if int(offs.max()) >= g.n_offsets:
            raise CorruptData("segment offset outside the block geometry")
    out = []
    for a, q in enumerate(split_codes(seg, offs, g)):                 # quantizer.py:250-272
        eb_int = inner_bound(h.eb_abs, mins[a], maxs[a], h.prec)
        out.append(_midpoints(q, mins[a], eb_int, h.prec).astype(_NPTYPE[h.prec]))
    if h.preserve:                                                    # pipeline.py:149-156
        ranks = unpack(raw[3], n, widths[3])
        if ranks.size and (int(ranks.max()) >= n or np.bincount(ranks.astype(np.int64)).max() > 1):
            raise CorruptData("rank stream is not a permutation")
        order = np.empty(n, np.int64)
        order[ranks.astype(np.int64)] = np.arange(n)
        out = [a[order] for a in out]
    return out


def decompress(data: bytes) -> list[np.ndarray]:
    """pipeline.decompress, pipeline.py:160-205 -> list of axis arrays."""
    h, table, payload = read_container(bytes(data))
    blocks = []
    for i in range(h.blocks):
        try:
            axes = decode_block(payload[int(table[i]):int(table[i + 1])], h)
            want = h.block_size if i + 1 < h.blocks else h.count - h.block_size * (h.blocks - 1)
            if axes[0].size != want:
                raise CorruptData(f"{axes[0].size} particles where the boundary math needs {want}")
        except OracleError as exc:
            raise CorruptData(f"block {i}: {exc}") from None
        blocks.append(axes)
    dt = _NPTYPE[h.prec]
    out = [np.concatenate([b[a] for b in blocks]) if blocks else np.empty(0, dt) for a in range(h.dims)]
    for i, a in enumerate(out):                                       # Dataset(...) model.py:75-77
        if a.size and not np.isfinite(a).all():
            raise DomainError(f"axis {i} contains non-finite coordinates")
    if out[0].size != h.count:
        raise CorruptData(f"blocks decode to {out[0].size} particles, header says {h.count}")
    return out


def iter_blocks(data: bytes):
    """iter_decompressed_blocks, pipeline.py:208-215."""
    h, table, payload = read_container(bytes(data))
    for i in range(h.blocks):
        try:
            yield decode_block(payload[int(table[i]):int(table[i + 1])], h)
        except OracleError as exc:
            raise CorruptData(f"block {i}: {exc}") from None


# --------------------------------------------------------------------------
# evaluation — block pairing, NRMSE, PSNR, bound check (metrics.py:49-200)


def block_order(block_axes, g: Geometry, eb_abs: float, prec: int) -> np.ndarray:
    """metrics._block_order, metrics.py:49-51: lexsort by (seg, offset, index)."""
    qs = [quantize_axis(a, g.mins[i], g.maxs[i], g.Q[i], eb_abs, prec) for i, a in enumerate(block_axes)]
    seg, off = linearize(qs, g)
    return np.lexsort((np.arange(seg.size), off, seg))


def pair_blocks(orig, rec, block_size: int, target: int, eb_abs: float):
    """metrics.pair_blocks, metrics.py:54-81 (eb_abs already resolved)."""
    orig, prec = check_axes(orig)
    rec = [np.asarray(a) for a in rec]
    if len(orig) != len(rec) or orig[0].size != rec[0].size:
        raise DomainError("datasets differ in shape, cannot pair")
    check_axes(rec)
    n = orig[0].size
    oi = np.empty(n, np.int64)
    ri = np.empty(n, np.int64)
    for start in range(0, n, block_size):
        sl = slice(start, min(start + block_size, n))
        ob = [a[sl] for a in orig]
        rb = [a[sl].astype(_NPTYPE[prec]) for a in rec]
        g = geometry([float(a.min()) for a in ob], [float(a.max()) for a in ob], eb_abs, target, prec)
        oi[sl] = start + block_order(ob, g, eb_abs, prec)
        ri[sl] = start + block_order(rb, g, eb_abs, prec)
    return oi, ri


def nrmse(o, r, pairing=None) -> float:
    """metrics.nrmse, metrics.py:84-104."""
    o = np.asarray(o, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    if pairing is not None:
        o = o[pairing[0]]
        r = r[pairing[1]]
    if o.size == 0:
        return 0.0
    rmse = math.sqrt(float(np.mean((o - r) ** 2)))
    span = float(o.max() - o.min())
    if span <= 0.0:
        if rmse == 0.0:
            return 0.0
        raise DomainError("degenerate field range with nonzero error")
    return rmse / span


def aggregate_psnr(values) -> float:
    """metrics.aggregate_psnr, metrics.py:107-119."""
    values = [float(v) for v in values]
    if not values:
        raise DomainError("aggregate PSNR of no fields")
    mean_sq = sum(v * v for v in values) / len(values)
    return math.inf if mean_sq == 0.0 else -20.0 * math.log10(math.sqrt(mean_sq))


def verify_bound(orig, rec, eb_abs: float, block_size: int, target: int):
    """metrics.verify_bound, metrics.py:131-152 -> (max_err, violations, checked)."""
    oi, ri = pair_blocks(orig, rec, block_size, target, eb_abs)
    max_err, viol = 0.0, []
    for a in range(len(orig)):
        d = np.abs(np.asarray(orig[a], np.float64)[oi] - np.asarray(rec[a], np.float64)[ri])
        if d.size:
            max_err = max(max_err, float(d.max()))
        viol.extend((a, int(oi[i]), float(d[i])) for i in np.flatnonzero(d > eb_abs))
    return max_err, viol, orig[0].size * len(orig)


# --------------------------------------------------------------------------
# synthetic generators (bench.py:56-94), used for fixtures


def gen_clusters(count, dims=3, seed=0, prec=F32, extent=1.0, clusters=32, sigma=0.01):
    """bench._gaussian_clusters, bench.py:60-70 (cluster-contiguous storage)."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(0.0, extent, size=(clusters, dims))
    base, extra = divmod(count, clusters)
    sizes = np.full(clusters, base, np.int64)
    sizes[:extra] += 1
    pts = centers[np.repeat(np.arange(clusters), sizes)] + rng.normal(0.0, sigma, size=(count, dims))
    return [np.ascontiguousarray(pts[:, a], dtype=_NPTYPE[prec]) for a in range(dims)]


def gen_uniform(count, dims=3, seed=0, prec=F32, extent=1.0):
    """bench._uniform_box, bench.py:56-57."""
    rng = np.random.default_rng(seed)
    return [rng.uniform(0.0, extent, count).astype(_NPTYPE[prec]) for _ in range(dims)]


def gen_lattice(count, dims=3, seed=0, prec=F32, pitch=0.05, jitter=0.01):
    """bench._jittered_lattice, bench.py:73-83."""
    rng = np.random.default_rng(seed)
    side = max(1, round(count ** (1.0 / dims)))
    while side ** dims < count:
        side += 1
    grids = np.meshgrid(*[np.arange(side, dtype=np.float64)] * dims, indexing="ij")
    out = []
    for gr in grids:
        flat = gr.reshape(-1)[:count] * pitch + rng.uniform(-jitter, jitter, count)
        out.append(flat.astype(_NPTYPE[prec]))
    return out
