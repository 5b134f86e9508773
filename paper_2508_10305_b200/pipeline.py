"""compress / decompress behind the reference's API, on the B200 kernels.

Mirrors ``gpz.pipeline`` (pipeline.py:32-215): same function names,
arguments, return types, error classes and "block {i}: ..." messages.  All
numeric work runs in ``_gpzb.so`` (include/gpzb.h) on the current CUDA
device and stream; this module only moves buffers and maps status codes.

Extra entry points for device-resident data (no host round trip):
``compress_device(ds_or_axes, cfg) -> torch.uint8 CUDA tensor`` and
``decompress_device(container_tensor) -> Dataset`` of CUDA tensors.
"""

from __future__ import annotations

import ctypes
import struct
import threading
from typing import Iterator

import numpy as np
import torch

from . import _lib
from ._lib import lib
from .errors import CorruptData, DomainError, GpzError, WidthOverflow
from .model import CompressConfig, Dataset, EbMode, Precision

__all__ = [
    "compress",
    "decompress",
    "compress_device",
    "compress_batch_device",
    "decompress_batch_device",
    "decompress_device",
    "iter_block_slices",
    "iter_decompressed_blocks",
    "resolve_absolute_bound",
    "parse_header",
]

# reason codes used for message shaping (gpzb_common.cuh)
_R_NONFINITE, _R_NONFINITE_OUT = 1, 60


_CUDA_OK = False


def _device() -> torch.device:
    global _CUDA_OK
    if not _CUDA_OK:  # checked once: torch.cuda.is_available() reads the environment on every call
        if not torch.cuda.is_available():
            raise RuntimeError("the GPZ B200 path needs a CUDA device (there is no CPU fallback)")
        _CUDA_OK = True
    return torch.device("cuda", torch.cuda.current_device())


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


# Every scratch buffer and helper stream is cached per *thread* (and device
# and slot): calls from different threads never share a workspace, a side
# buffer, a pinned staging buffer or a stream, so concurrent compress /
# decompress calls on distinct data are safe, as the reference's pure
# functions are.
_TLS = threading.local()


def _tls(name: str) -> dict:
    d = getattr(_TLS, name, None)
    if d is None:
        d = {}
        setattr(_TLS, name, d)
    return d


def _workspace(nbytes: int, slot: int = 0) -> torch.Tensor:
    """Per-thread, per-device scratch, grown on demand (the library never
    allocates); one buffer per concurrent slot (compress_batch_device)."""
    dev = _device()
    cache = _tls("ws")
    key = (dev.index, slot)
    buf = cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, device=dev)
        cache[key] = buf
    return buf


def _side(slot: int, nbytes: int = 0) -> torch.Tensor:
    """Side buffer for the general encoder's payloads (K2w), cached like the
    workspace; it only grows when a compression reports GPZB_NEED_SIDE."""
    dev = _device()
    cache = _tls("side")
    key = (dev.index, slot)
    buf = cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
        cache[key] = buf
    return buf


def _check(st: int, res: "_lib.Result | None" = None) -> None:
    if st == _lib.OK:
        return
    if res is None:
        res = _lib.Result(status=st, reason=0, block=-1, axis=-1)
    msg = _lib.reason_message(res.reason)
    where = f"block {res.block}: " if res.block >= 0 else ""
    if st == _lib.DOMAIN:
        if res.reason in (_R_NONFINITE, _R_NONFINITE_OUT):
            raise DomainError(f"axis {res.axis} contains non-finite coordinates")
        raise DomainError(where + msg)
    if st == _lib.WIDTH:
        raise WidthOverflow(f"{where}axis {res.axis}: {msg}" if res.reason == 3 else where + msg)
    if st == _lib.CORRUPT:
        if res.axis >= 0 and res.reason in (33, 34, 35, 45, 46):
            msg = f"axis {res.axis}: {msg}"
        raise CorruptData(where + msg)
    if st == _lib.UNSUPPORTED:
        raise NotImplementedError(msg if res.reason else "configuration outside the CUDA kernels' envelope "
                                  f"(block_size <= {_lib.MAX_BLOCK_SIZE})")
    if st == _lib.INVALID:
        raise ValueError("invalid argument to the GPZ CUDA library")
    raise RuntimeError(f"CUDA error {st - 100} in the GPZ library")


def iter_block_slices(count: int, block_size: int) -> Iterator[slice]:
    """Storage-order block boundaries; the last block may be partial (pipeline.py:32-35)."""
    for start in range(0, count, block_size):
        yield slice(start, min(start + block_size, count))


def _as_dataset(ds) -> Dataset:
    if isinstance(ds, Dataset):
        return ds
    return Dataset.from_axes(list(ds))


def _device_axes(ds: Dataset) -> list:
    dev = _device()
    out = []
    for a in ds.axes:
        if isinstance(a, torch.Tensor):
            t = a if (a.is_cuda and a.device == dev) else a.to(dev, non_blocking=True)
        else:
            t = torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=False)
        out.append(t.contiguous())
    return out


class _Job:
    """One dataset's compression in flight (the phases of compress_device)."""

    __slots__ = ("axes", "ptrs", "count", "dims", "prec", "bs", "t", "pres", "eb", "mode", "ws", "out", "bound",
                 "nb", "res", "stream", "timing", "slot", "words")


def _ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def _compress_begin(ds, cfg: CompressConfig, slot: int, timing, plan: bool = True) -> _Job:
    """Allocate and enqueue the workspace reset, K1 and K1.5 (no host sync).
    plan=False stops after K1 (sharded runs reduce the range words first)."""
    j = _Job()
    ds = _as_dataset(ds)
    j.axes = _device_axes(ds)
    j.count, j.dims, j.prec = ds.count, ds.dims, ds.precision.value
    j.bs, j.t, j.pres = cfg.block_size, cfg.target_segs_per_axis, int(cfg.preserve_order)
    j.eb, j.mode = float(cfg.error_bound), cfg.eb_mode.value
    j.timing = timing
    j.slot, j.words = slot, None
    ws_bytes = ctypes.c_uint64()
    _check(lib.gpzb_compress_workspace(j.count, j.dims, j.prec, j.bs, ctypes.byref(ws_bytes)))
    bound = ctypes.c_uint64()
    _check(lib.gpzb_compress_bound(j.count, j.dims, j.prec, j.bs, j.t, j.pres, ctypes.byref(bound)))
    j.bound = bound.value
    j.ws = _workspace(ws_bytes.value, slot)
    j.out = None  # allocated at its exact size once the scan has run (_compress_finish)
    j.ptrs = _lib.ptr_array([a.data_ptr() for a in j.axes])
    j.res = _lib.Result()
    j.stream = _stream()
    j.nb = (j.count + j.bs - 1) // j.bs
    if j.count == 0:
        return j
    _check(lib.gpzb_workspace_reset_async(j.ws.data_ptr(), j.ws.numel(), j.count, j.bs, j.stream))
    e0 = _ev() if timing is not None else None
    _check(lib.gpzb_range_async(j.ptrs, j.dims, j.prec, j.count, j.bs, j.ws.data_ptr(), j.ws.numel(), j.stream))
    if timing is not None:
        timing.setdefault("range", []).append((e0, _ev()))
    if plan:
        _compress_plan(j)
    return j


def _compress_plan(j: _Job) -> None:
    """Enqueue K1.5 (bound resolution from the range words + block routing)."""
    if j.count:
        _check(lib.gpzb_encode_plan_async(j.ptrs, j.dims, j.prec, j.count, j.eb, j.mode, j.bs, j.t, j.pres,
                                          j.ws.data_ptr(), j.ws.numel(), j.stream))


def _compress_encode(j: _Job) -> None:
    """Enqueue the encoders + K3 (no host sync: every encoder reads its block
    count on the device)."""
    if j.count == 0:
        return
    side = _side(j.slot)
    e0 = _ev() if j.timing is not None else None
    _check(lib.gpzb_encode_async(j.ptrs, j.dims, j.prec, j.count, j.eb, j.mode, j.bs, j.t, j.pres, j.ws.data_ptr(),
                                 j.ws.numel(), side.data_ptr(), side.numel(), None, 0, 0,
                                 j.count, j.nb, 1, j.stream))
    if j.timing is not None:
        j.timing.setdefault("encode", []).append((e0, None))


def _compress_emit(j: _Job, table_base: int = 0, header_count=None, header_blocks=None,
                   write_header: int = 1) -> torch.Tensor:
    """After a successful result read: allocate the container at its exact
    size and enqueue K3b (offset table, header, payload moves) into it."""
    j.out = torch.empty(j.res.out_len, dtype=torch.uint8, device=j.axes[0].device)
    side = _side(j.slot)
    _check(lib.gpzb_emit_async(j.ptrs, j.dims, j.prec, j.count, j.eb, j.mode, j.bs, j.pres, j.ws.data_ptr(),
                               j.ws.numel(), side.data_ptr(), j.out.data_ptr(), j.out.numel(), table_base,
                               j.count if header_count is None else header_count,
                               j.nb if header_blocks is None else header_blocks, write_header, j.stream))
    if j.timing is not None and j.timing.get("encode") and j.timing["encode"][-1][1] is None:
        j.timing["encode"][-1] = (j.timing["encode"][-1][0], _ev())
    return j.out


def _compress_status(j: _Job) -> int:
    """Read the result record (one sync of the job's stream); no raising.
    When general-encoder blocks outgrew the cached side buffer the library
    wrote nothing for them and reports the size: grow it and encode again
    (the range words of a sharded run are restored from j.words)."""
    if j.count == 0:
        j.out = torch.empty(j.bound, dtype=torch.uint8, device=j.axes[0].device)
        return lib.gpzb_compress(j.ptrs, j.dims, j.prec, j.count, j.eb, j.mode, j.bs, j.t, j.pres, j.ws.data_ptr(),
                                 j.ws.numel(), j.out.data_ptr(), j.bound, j.stream, ctypes.byref(j.res))
    st = lib.gpzb_compress_result(j.ws.data_ptr(), j.ws.numel(), j.count, j.bs, j.stream, ctypes.byref(j.res))
    if st == _lib.NEED_SIDE:
        _side(j.slot, j.res.side_bytes)
        with torch.cuda.stream(torch.cuda.ExternalStream(j.stream)):
            _check(lib.gpzb_workspace_reset_async(j.ws.data_ptr(), j.ws.numel(), j.count, j.bs, j.stream))
            _check(lib.gpzb_range_async(j.ptrs, j.dims, j.prec, j.count, j.bs, j.ws.data_ptr(), j.ws.numel(),
                                        j.stream))
            if j.words is not None:
                j.ws[40:56].view(torch.int64).copy_(j.words)
            _compress_plan(j)
            timing, j.timing = j.timing, None
            _compress_encode(j)
            j.timing = timing
        st = lib.gpzb_compress_result(j.ws.data_ptr(), j.ws.numel(), j.count, j.bs, j.stream, ctypes.byref(j.res))
    return st


def _remember_header(t: torch.Tensor, j: _Job) -> torch.Tensor:
    """Attach the container's parsed global header to the returned tensor, so
    that decompressing it again skips the header's device-to-host read (and
    the stream sync it costs) while the tensor is unmodified (torch's version
    counter) — the same fields K3b wrote (container.py:84-95)."""
    head = struct.pack("<4sHBBBBddIQQ", b"GPZ1", 1, j.dims, j.prec, j.pres, j.mode, j.eb, j.res.eb_abs, j.bs,
                       j.count, j.nb)
    t._gpzb_header = (parse_header(head, t.numel()), t._version, t.data_ptr(), t.numel())
    return t


def _known_header(t: torch.Tensor):
    k = getattr(t, "_gpzb_header", None)
    if k is not None and k[1] == t._version and k[2] == t.data_ptr() and k[3] == t.numel():
        return k[0]
    return None


def _compress_finish(j: _Job) -> torch.Tensor:
    """Read the result record (one sync) and map errors."""
    st = _compress_status(j)
    _check(st, j.res)
    compress_device.last_result = j.res
    _tls("last").update(ws=j.ws, count=j.count, bs=j.bs, dims=j.dims, prec=j.prec)
    if j.count == 0:
        return j.out[: j.res.out_len].clone()
    return _remember_header(_compress_emit(j), j)


def last_path_counts() -> list:
    """Diagnostics: blocks per encoder path of this thread's last compression
    (include/gpzb.h gpzb_encode_path_counts)."""
    c = (ctypes.c_uint64 * 8)()
    w = _tls("last")
    _check(lib.gpzb_encode_path_counts(w["ws"].data_ptr(), w["ws"].numel(), w["count"], w["bs"], w["dims"],
                                       w["prec"], _stream(), c))
    return list(c)


def compress_device(ds, cfg: CompressConfig, *, timing=None) -> torch.Tensor:
    """Container bytes as a CUDA uint8 tensor (a view of the output buffer).

    ``timing``: optional dict; when given, CUDA events are recorded on the
    current stream around the range kernel (K1) and the encode call (K2 +
    K3) and appended to ``timing["range"]`` / ``timing["encode"]`` as pairs.
    """
    j = _compress_begin(ds, cfg, 0, timing)
    _compress_encode(j)
    return _compress_finish(j)


def _side_stream(i: int) -> torch.cuda.Stream:
    """Stream i of the batched calls (per thread): earlier datasets get higher
    priority, so the first range pass finishes first and its encoder starts
    while the next range pass still streams (a pipeline instead of two halves
    contending)."""
    dev = _device()
    streams = _tls("streams")
    key = (dev.index, i)
    if key not in streams:
        lo, hi = torch.cuda.Stream.priority_range()  # (lowest, highest); higher priority = smaller number
        streams[key] = torch.cuda.Stream(device=dev, priority=max(hi, min(lo, hi + i)))
    return streams[key]


def compress_batch_device(datasets, cfg: CompressConfig, *, timing=None) -> list:
    """Compress several datasets (e.g. the position and velocity fields of one
    snapshot) with one CUDA stream and workspace each, so the HBM-bound range
    pass (K1) of one overlaps the compute-bound encoder (K2) of another.
    Returns the containers in order; each is byte-identical to compress_device."""
    cur = torch.cuda.current_stream()
    start = torch.cuda.Event()
    start.record(cur)
    jobs = []
    for i, ds in enumerate(datasets):
        s = _side_stream(i)
        s.wait_event(start)
        with torch.cuda.stream(s):
            jobs.append(_compress_begin(ds, cfg, i, timing))
    # the encoders run one dataset at a time (job i's waits for job i-1's):
    # two compute-bound encoders sharing the SMs finish later than the two in
    # sequence; only the HBM-bound range passes overlap an encoder
    prev = None
    for i, j in enumerate(jobs):
        s = _side_stream(i)
        if prev is not None:
            s.wait_event(prev)
        with torch.cuda.stream(s):
            _compress_encode(j)
            prev = torch.cuda.Event()
            prev.record(s)
    outs = []
    for i, j in enumerate(jobs):
        s = _side_stream(i)
        with torch.cuda.stream(s):
            outs.append(_compress_finish(j))
        cur.wait_stream(s)
        outs[-1].record_stream(cur)
    return outs


def _pinned(nbytes: int) -> torch.Tensor:
    """This thread's pinned host staging buffer (grown on demand)."""
    cache = _tls("pinned")
    buf = cache.get("out")
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        cache["out"] = buf
    return buf


_api = ctypes.pythonapi
_api.PyBytes_FromStringAndSize.restype = ctypes.py_object
_api.PyBytes_FromStringAndSize.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
try:
    _libc = ctypes.CDLL(None)
    _libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
except (OSError, AttributeError):  # pragma: no cover
    _libc = None
_MADV_HUGEPAGE = 14
_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        import concurrent.futures
        import os

        _POOL = concurrent.futures.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1))
    return _POOL


def _memmove_parts(dst: int, src: int, n: int, futs: list) -> None:
    """Queue a memmove split over the host threads (ctypes releases the GIL)."""
    pool = _pool()
    step = max(4 << 20, (n + pool._max_workers - 1) // pool._max_workers)
    futs.extend(pool.submit(ctypes.memmove, dst + o, src + o, min(step, n - o)) for o in range(0, n, step))


def _par_memmove(dst: int, src: int, n: int) -> None:
    if n < (32 << 20):
        ctypes.memmove(dst, src, n)
        return
    futs: list = []
    _memmove_parts(dst, src, n, futs)
    for f in futs:
        f.result()


_CHUNK = 64 << 20  # host <-> device pipelining granule


def _device_to_bytes(t: torch.Tensor) -> bytes:
    """A fresh ``bytes`` object holding a device buffer.  The D2H runs in
    64 MiB chunks into a cached pinned buffer; each chunk is moved into the
    bytes storage by the host threads as soon as its copy lands, so the PCIe
    copy and the host copy (and its first-touch page faults, 2 MiB ones:
    the storage is advised to transparent huge pages) overlap."""
    n = t.numel()
    host = _pinned(n)[:n]
    b = _api.PyBytes_FromStringAndSize(None, n)
    addr = ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p).value
    if _libc is not None and n >= (4 << 20):
        hp = 2 << 20
        s0, s1 = (addr + hp - 1) & ~(hp - 1), (addr + n) & ~(hp - 1)
        if s1 > s0:
            _libc.madvise(s0, s1 - s0, _MADV_HUGEPAGE)
    if n < 2 * _CHUNK:
        host.copy_(t)
        _par_memmove(addr, host.data_ptr(), n)
        return b
    stream = torch.cuda.current_stream(t.device)
    evs = []
    for o in range(0, n, _CHUNK):
        host[o: o + _CHUNK].copy_(t[o: o + _CHUNK], non_blocking=True)
        e = torch.cuda.Event()
        e.record(stream)
        evs.append((o, min(_CHUNK, n - o), e))
    futs: list = []
    for o, m, e in evs:
        e.synchronize()
        _memmove_parts(addr + o, host.data_ptr() + o, m, futs)
    for f in futs:
        f.result()
    return b


def compress(ds: Dataset, cfg: CompressConfig, workers: int = 1) -> bytes:
    """Compress a dataset into container bytes, deterministically (pipeline.py:73-103).

    ``workers`` is accepted for API compatibility; the output never depends
    on it (pipeline.py:6-7) and the GPU kernels ignore it.
    """
    del workers
    return _device_to_bytes(compress_device(ds, cfg))


def _host_bytes(data) -> np.ndarray:
    if isinstance(data, np.ndarray):
        return np.ascontiguousarray(data.view(np.uint8).reshape(-1))
    return np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8)


def parse_header(head: bytes, container_len: int) -> _lib.Header:
    """read_container's global-header checks (container.py:245-281), in C."""
    h = _lib.Header()
    res = _lib.Result()
    buf = bytes(head[: _lib.GLOBAL_HEADER_SIZE])
    st = lib.gpzb_parse_header(buf, len(buf), container_len, ctypes.byref(h), ctypes.byref(res))
    _check(st, res)
    return h


def _to_device_bytes(data) -> tuple[torch.Tensor, _lib.Header]:
    if isinstance(data, torch.Tensor):
        known = _known_header(data) if data.is_cuda else None
        if known is not None:  # compress_device's own 1-D uint8 result
            return data, known
        t = data.reshape(-1).view(torch.uint8)
        if not t.is_cuda:
            t = t.to(_device(), non_blocking=True)
        head = t[: _lib.GLOBAL_HEADER_SIZE].cpu().numpy().tobytes()
        return t, parse_header(head, t.numel())
    host = _host_bytes(data)
    h = parse_header(host[: _lib.GLOBAL_HEADER_SIZE].tobytes(), host.size)
    # threaded copies into the cached pinned buffer, 64 MiB at a time, each
    # chunk's H2D queued as soon as it is staged (host and PCIe copies overlap)
    n = host.size
    stage = _pinned(n)[:n]
    t = torch.empty(n, dtype=torch.uint8, device=_device())
    for o in range(0, n, _CHUNK):
        m = min(_CHUNK, n - o)
        _par_memmove(stage.data_ptr() + o, host.ctypes.data + o, m)
        t[o: o + m].copy_(stage[o: o + m], non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()  # the stage is reused by the next call
    return t, h


def _decode_launch(t: torch.Tensor, h: _lib.Header, offsets=None, capacity=None, timing=None, slot: int = 0,
                   stream: int | None = None):
    """Enqueue K4a + K4w + the list decoder; returns what _decode_result needs
    (the output views are cut after the launch: the GPU starts sooner)."""
    if capacity is None:
        capacity = min(h.particle_count, h.block_count * min(h.block_size, _lib.MAX_BLOCK_SIZE))
    # one allocation for every axis (rows 16-byte aligned), one allocator call
    cap1 = max(capacity, 1)
    row = (cap1 + 3) & ~3
    big = torch.empty(h.dims * row, dtype=_DTYPES[h.precision], device=t.device)
    base, rb = big.data_ptr(), row * big.element_size()
    wkey = (h.block_count, h.block_size)
    wcache = _tls("dec_ws_bytes")
    ws_bytes = wcache.get(wkey)
    if ws_bytes is None:
        v = ctypes.c_uint64()
        _check(lib.gpzb_decompress_workspace(ctypes.byref(h), ctypes.byref(v)))
        ws_bytes = wcache[wkey] = v.value
    ws = _workspace(ws_bytes, slot)
    if stream is None:
        stream = _stream()
    e0 = _ev() if timing is not None else None
    _check(lib.gpzb_decompress_async(t.data_ptr(), t.numel(), ctypes.byref(h),
                                     _lib.ptr_array([base + a * rb for a in range(h.dims)]), capacity,
                                     offsets.data_ptr() if offsets is not None else None, ws.data_ptr(),
                                     ws.numel(), stream))
    if timing is not None:
        timing.setdefault("decode", []).append((e0, _ev()))
    outs = [big[a * row: a * row + cap1] for a in range(h.dims)]
    return outs, ws, h, capacity


_DTYPES = {p.value: p.torch_dtype for p in Precision}


def _decode_result(launched, stream: int | None = None):
    outs, ws, h, capacity = launched
    res = _lib.Result()
    lib.gpzb_decompress_result(ws.data_ptr(), ws.numel(), ctypes.byref(h), _stream() if stream is None else stream,
                               ctypes.byref(res))
    return outs, res, capacity


def _decode(t: torch.Tensor, h: _lib.Header, offsets=None, capacity=None, timing=None):
    return _decode_result(_decode_launch(t, h, offsets, capacity, timing))


def decompress_batch_device(containers, *, timing=None) -> list:
    """Decode several containers with one CUDA stream and workspace each
    (overlapping their kernels); returns Datasets of CUDA tensors in order.
    The host work is arranged around the GPU's: every decode is enqueued
    before any output view or Dataset is built, and those are built before
    the first result read, so little host time is left on the critical path
    at either end of the call."""
    cur = torch.cuda.current_stream()
    start = torch.cuda.Event()
    start.record(cur)
    launched, streams = [], []
    for i, data in enumerate(containers):
        s = _side_stream(i)
        s.wait_event(start)
        known = _known_header(data) if isinstance(data, torch.Tensor) and data.is_cuda else None
        if known is not None:
            t, h = data, known
        else:
            with torch.cuda.stream(s):
                t, h = _to_device_bytes(data)
        # outputs are allocated on `cur` (the caller's stream): cur waits for s
        # below before anything on it can touch them
        launched.append(_decode_launch(t, h, timing=timing, slot=i, stream=s.cuda_stream))
        streams.append(s)
    out = []
    for s, (outs, _, h, _) in zip(streams, launched):
        cur.wait_stream(s)
        n = h.particle_count
        out.append(Dataset._trusted(tuple(o if o.numel() == n else o[:n] for o in outs), Precision(h.precision)))
    for s, L in zip(streams, launched):
        _, res, _ = _decode_result(L, s.cuda_stream)
        _check(res.status, res)
    return out


def _copy_stream(i: int = 0) -> torch.cuda.Stream:
    dev = _device()
    streams = _tls("copy_streams")
    st = streams.get((dev.index, i))
    if st is None:
        st = streams[(dev.index, i)] = torch.cuda.Stream(device=dev)
    return st


def _streamed_plan(host: np.ndarray, h: _lib.Header):
    """Block ranges for a chunked decode of a host container, or None when the
    container is small or its offset table is not well formed (the one-shot
    path then reports the reference's error for it)."""
    nb = h.block_count
    n = host.size
    if (nb < 2 or h.particle_count == 0 or n < (32 << 20) or h.table_end + h.payload_len != n
            or h.block_size > _lib.MAX_BLOCK_SIZE):
        return None
    # the output buffers are sized from particle_count: only trust it when it
    # agrees with the block count (else the one-shot decode reports the
    # reference's "block i: ... boundary" error, pipeline.py:174-181)
    if not (nb - 1) * h.block_size < h.particle_count <= nb * h.block_size:
        return None
    tab = host[_lib.GLOBAL_HEADER_SIZE: _lib.GLOBAL_HEADER_SIZE + 8 * (nb + 1)].view("<u8")
    if int(tab[0]) != 0 or int(tab[-1]) != h.payload_len or bool(np.any(tab[1:] < tab[:-1])):
        return None
    # chunks balanced by blocks (the axes' D2H dominates), at least 16 so the
    # last chunk's copy-out is a small tail, and at most _CHUNK payload bytes each
    k = max(16, -(-h.payload_len // _CHUNK))
    cuts = sorted(set(int(c) for c in np.linspace(0, nb, min(k, nb) + 1).round()))
    return tab, list(zip(cuts[:-1], cuts[1:]))


def _decode_streamed(host: np.ndarray, h: _lib.Header, plan, to_host: bool) -> Dataset:
    """decompress of a host container with the copies pipelined: chunk k's
    bytes are staged into pinned memory (host threads) and sent while chunk
    k-1 decodes (gpzb_decompress_range_async) and chunk k-2's particles go
    back to pinned host memory on a second stream.  The outcome (errors in
    the reference's precedence) is that of one decode over all blocks."""
    tab, chunks = plan
    n = host.size
    prec = Precision(h.precision)
    dev = _device()
    count, bs = h.particle_count, h.block_size
    capacity = min(count, h.block_count * min(bs, _lib.MAX_BLOCK_SIZE))
    outs = [torch.empty(capacity, dtype=prec.torch_dtype, device=dev) for _ in range(h.dims)]
    ptrs = _lib.ptr_array([o.data_ptr() for o in outs])
    ws_bytes = ctypes.c_uint64()
    _check(lib.gpzb_decompress_workspace(ctypes.byref(h), ctypes.byref(ws_bytes)))
    ws = _workspace(ws_bytes.value, 0)
    stage = _pinned(n)[:n]
    t = torch.empty(n, dtype=torch.uint8, device=dev)
    cur = torch.cuda.current_stream(dev)
    main = _copy_stream(1)  # upload + decode (a stream of its own: see DESIGN.md §8)
    main.wait_stream(cur)
    cs = _copy_stream(0) if to_host else None
    houts = [torch.empty(count, dtype=prec.torch_dtype, pin_memory=True) for _ in range(h.dims)] if to_host else None
    if cs is not None:
        cs.wait_stream(main)
    done = 0
    for k, (b0, b1) in enumerate(chunks):
        end = n if b1 == h.block_count else h.table_end + int(tab[b1])
        if end > done:
            _par_memmove(stage.data_ptr() + done, host.ctypes.data + done, end - done)
            with torch.cuda.stream(main):
                t[done:end].copy_(stage[done:end], non_blocking=True)
            done = end
        _check(lib.gpzb_decompress_range_async(t.data_ptr(), n, ctypes.byref(h), ptrs, capacity, None,
                                               ws.data_ptr(), ws.numel(), b0, b1, int(k == 0), main.cuda_stream))
        if cs is not None:
            e = torch.cuda.Event()
            e.record(main)
            cs.wait_event(e)
            p0, p1 = b0 * bs, min(b1 * bs, count)
            with torch.cuda.stream(cs):
                for ho, o in zip(houts, outs):
                    ho[p0:p1].copy_(o[p0:p1], non_blocking=True)
    res = _lib.Result()
    lib.gpzb_decompress_result(ws.data_ptr(), ws.numel(), ctypes.byref(h), main.cuda_stream, ctypes.byref(res))
    if cs is not None:
        cs.synchronize()
    cur.wait_stream(main)  # (main is already idle: gpzb_decompress_result synchronised it)
    _check(res.status, res)
    if to_host:
        return Dataset(axes=tuple(o.numpy() for o in houts), precision=prec)
    return Dataset(axes=tuple(o[:count] for o in outs), precision=prec)


def _streamed(data, to_host: bool):
    """(_decode_streamed result) for host bytes-like containers, else None."""
    if isinstance(data, torch.Tensor):
        return None
    host = _host_bytes(data)
    if host.size < (32 << 20):
        return None
    h = parse_header(host[: _lib.GLOBAL_HEADER_SIZE].tobytes(), host.size)
    plan = _streamed_plan(host, h)
    if plan is None:
        return None
    return _decode_streamed(host, h, plan, to_host)


def decompress_device(data, workers: int = 1, *, header=None, timing=None) -> Dataset:
    """Reconstruct on the GPU; the returned Dataset holds CUDA tensors.

    ``header``: an already parsed header (skips the 46-byte read-back);
    ``timing``: optional dict receiving CUDA event pairs around K4."""
    del workers
    if header is not None and isinstance(data, torch.Tensor) and data.is_cuda:
        t, h = data, header
    elif timing is None and (ds := _streamed(data, to_host=False)) is not None:
        return ds
    else:
        t, h = _to_device_bytes(data)
    outs, res, _ = _decode(t, h, timing=timing)
    _check(res.status, res)
    n = h.particle_count
    return Dataset(axes=tuple(o[:n] for o in outs), precision=Precision(h.precision))


def decompress(data, workers: int = 1) -> Dataset:
    """Reconstruct a dataset from container bytes (pipeline.py:160-205).

    Particles come back in sorted intra-block order unless the container
    preserves order; block boundaries always match the original.  The axes
    are numpy arrays over pinned host memory (PyTorch's caching host
    allocator).  Containers of 32 MiB and more are decoded in chunks of
    blocks so that the container's upload, the decode and the particles'
    download overlap (_decode_streamed).
    """
    ds = _streamed(data, to_host=True)
    if ds is not None:
        return ds
    ds = decompress_device(data, workers)
    outs = [torch.empty(a.numel(), dtype=a.dtype, pin_memory=True) for a in ds.axes]
    for o, a in zip(outs, ds.axes):
        o.copy_(a, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return Dataset(axes=tuple(o.numpy() for o in outs), precision=ds.precision)


def iter_decompressed_blocks(data) -> Iterator[list]:
    """Per-block reconstructed axes (pipeline.py:208-215): the blocks before
    the first corrupt one are yielded, then CorruptData("block i: ...")."""
    t, h = _to_device_bytes(data)
    if h.block_count == 0:
        return
    counts = torch.zeros(h.block_count, dtype=torch.int64, device=t.device)
    _check(lib.gpzb_block_counts_async(t.data_ptr(), t.numel(), ctypes.byref(h), counts.data_ptr(), _stream()))
    offsets = torch.zeros_like(counts)
    offsets[1:] = torch.cumsum(counts, 0)[:-1]
    capacity = int(counts.sum().item())
    outs, res, _ = _decode(t, h, offsets, capacity)
    if res.table_flags:
        _check(res.status, res)
    stop = res.decode_block if res.decode_block >= 0 else h.block_count
    host = [o[:capacity].cpu().numpy() for o in outs]
    cnt = counts.cpu().numpy()
    off = offsets.cpu().numpy()
    for i in range(stop):
        yield [a[off[i]: off[i] + cnt[i]].copy() for a in host]
    if res.decode_block >= 0:
        r = _lib.Result(status=_lib.CORRUPT, reason=res.decode_reason, block=res.decode_block,
                        axis=res.decode_axis)
        st = _lib.UNSUPPORTED if res.decode_reason in (53, 70) else _lib.CORRUPT
        _check(st, r)


def _ukey_inv(k: int) -> float:
    b = (k & 0x7FFFFFFFFFFFFFFF) if (k >> 63) else (~k & 0xFFFFFFFFFFFFFFFF)
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def resolve_absolute_bound(ds: Dataset, cfg: CompressConfig) -> float:
    """model.resolve_absolute_bound (model.py:183-199); the joint range comes
    from the range kernel K1 on the GPU."""
    if cfg.eb_mode is EbMode.ABSOLUTE:
        return float(cfg.error_bound)
    ds = _as_dataset(ds)
    if ds.count == 0:
        raise DomainError("range-relative bound is undefined for an empty dataset")
    axes = _device_axes(ds)
    bs = min(cfg.block_size, _lib.CTA_BLOCK_SIZE)  # the joint range does not depend on the block size
    ws_bytes = ctypes.c_uint64()
    _check(lib.gpzb_compress_workspace(ds.count, ds.dims, ds.precision.value, bs, ctypes.byref(ws_bytes)))
    ws = _workspace(ws_bytes.value)
    _check(lib.gpzb_workspace_reset_async(ws.data_ptr(), ws.numel(), ds.count, bs, _stream()))
    _check(lib.gpzb_range_async(_lib.ptr_array([a.data_ptr() for a in axes]), ds.dims, ds.precision.value,
                                ds.count, bs, ws.data_ptr(), ws.numel(), _stream()))
    head = ws[:64].cpu().numpy()
    nonfinite = int(head[16:20].view(np.uint32)[0])
    if nonfinite:
        axis = (nonfinite & -nonfinite).bit_length() - 1
        raise DomainError(f"axis {axis} contains non-finite coordinates")
    w0, w1 = (int(v) for v in head[40:56].view(np.uint64))
    lo, hi = -_ukey_inv(w0), _ukey_inv(w1)
    span = hi - lo
    if span <= 0.0:
        span = 1.0
    return float(cfg.error_bound) * span
