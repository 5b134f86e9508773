"""``.gpz`` files and random block access.

The container format is the reference's (container.py:3-23): 46-byte global
header, (B+1) little-endian u64 payload offsets, payloads.  Because block i
occupies payload bytes [table[i], table[i+1]), any block range can be
decoded from three small reads: the header, B'+1 table entries and the
payload span — no full-file read, no full decode.

* ``write_container(path, data)`` / ``read_container(path)`` — whole
  containers between files and host bytes or HBM (pinned, chunked copies).
* ``write_sharded(path, sc)`` — every rank of a sharded compression
  (sharded.py) writes its own table slice and payload at their global file
  offsets (``os.pwrite``); rank 0 writes the header.  Nothing is gathered.
* ``decompress_blocks(src, first, last)`` — reconstruct blocks
  [first, last) of a container held in bytes, a CUDA tensor or a file;
  ``iter_file_blocks(path, chunk)`` streams a file chunk by chunk.

``sub_container`` is the pure host step shared by both: it rebases a table
slice into a self-contained container of the block range (the reference's
decoder semantics apply unchanged; the errors' block indices are shifted
back to the original numbering).
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .errors import CorruptData

__all__ = ["write_container", "read_container", "write_sharded", "sub_container", "decompress_blocks",
           "iter_file_blocks", "HEADER_FMT"]

HEADER_FMT = "<4sHBBBBddIQQ"  # container.py:57
HEADER_SIZE = 46
_CHUNK = 64 << 20


def _is_path(src) -> bool:
    return isinstance(src, (str, os.PathLike))


def write_container(path, data) -> int:
    """Write a container (bytes-like, numpy, or CUDA/CPU uint8 tensor) to
    ``path``; returns the byte count.  Device data moves in 64 MiB chunks
    through one pinned buffer."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    with open(path, "wb") as f:
        if torch is not None and isinstance(data, torch.Tensor):
            t = data.reshape(-1).view(torch.uint8)
            if not t.is_cuda:
                f.write(t.numpy().tobytes())
                return t.numel()
            pin = torch.empty(min(_CHUNK, max(t.numel(), 1)), dtype=torch.uint8, pin_memory=True)
            for s in range(0, t.numel(), _CHUNK):
                e = min(s + _CHUNK, t.numel())
                pin[: e - s].copy_(t[s:e])
                f.write(memoryview(pin.numpy())[: e - s])
            return t.numel()
        mv = memoryview(data).cast("B")
        f.write(mv)
        return mv.nbytes


def read_container(path, device: bool = False):
    """The file's bytes (``device=False``) or a CUDA uint8 tensor with them."""
    if not device:
        with open(path, "rb") as f:
            return f.read()
    import torch

    from .pipeline import _device

    size = os.path.getsize(path)
    out = torch.empty(size, dtype=torch.uint8, device=_device())
    pin = torch.empty(min(_CHUNK, max(size, 1)), dtype=torch.uint8, pin_memory=True)
    with open(path, "rb", buffering=0) as f:
        for s in range(0, size, _CHUNK):
            e = min(s + _CHUNK, size)
            n = f.readinto(memoryview(pin.numpy())[: e - s])
            if n != e - s:
                raise CorruptData("file shrank while reading")
            out[s:e].copy_(pin[: e - s])  # synchronous: the pinned buffer is reused next round
    return out


def write_sharded(path, sc) -> None:
    """Collective over the default process group: the global container of a
    sharded compression, written in place by every rank (no gather)."""
    import torch.distributed as dist

    from .sharded import global_pieces

    t_off, tbytes, p_off, payload = global_pieces(sc)
    total = HEADER_SIZE + 8 * (sc.global_blocks + 1) + sc.global_payload
    if sc.rank == 0:
        with open(path, "wb") as f:
            f.truncate(total)
            f.write(sc.header)
    dist.barrier()
    fd = os.open(path, os.O_WRONLY)
    try:
        for off, buf in ((t_off, tbytes), (p_off, payload)):
            mv = memoryview(buf)
            while mv.nbytes:
                n = os.pwrite(fd, mv, off)
                mv, off = mv[n:], off + n
    finally:
        os.close(fd)
    dist.barrier()


def _header_fields(head: bytes):
    (magic, version, dims, prec, flags, mode, eb, eb_abs, bs, count, blocks) = struct.unpack(HEADER_FMT, head)
    return dict(magic=magic, version=version, dims=dims, prec=prec, flags=flags, mode=mode, eb=eb,
                eb_abs=eb_abs, bs=bs, count=count, blocks=blocks)


def sub_container(head: bytes, table: np.ndarray, payload, first: int, last: int) -> bytes:
    """Self-contained container of blocks [first, last) of a container with
    global header ``head``: ``table`` holds its entries first..last
    (last - first + 1 values), ``payload`` the bytes [table[0], table[-1])
    of its payload region."""
    h = _header_fields(head)
    nb = last - first
    if last < h["blocks"]:
        count = nb * h["bs"]
    else:
        count = max(0, h["count"] - first * h["bs"])
    t = np.asarray(table, dtype=np.uint64)
    rebased = (t - t[0]).astype("<u8")
    new_head = struct.pack(HEADER_FMT, h["magic"], h["version"], h["dims"], h["prec"], h["flags"], h["mode"],
                           h["eb"], h["eb_abs"], h["bs"], count, nb)
    return new_head + rebased.tobytes() + bytes(payload)


def _read_range(src, first: int, last: int):
    """(header, table entries first..last, payload span) from bytes / tensor / file."""
    if _is_path(src):
        fd = os.open(src, os.O_RDONLY)
        try:
            size = os.fstat(fd).st_size
            head = os.pread(fd, HEADER_SIZE, 0)
            if len(head) < HEADER_SIZE:
                raise CorruptData("container shorter than the 46-byte global header")
            h = _header_fields(head)
            _check_range(h, first, last)
            traw = os.pread(fd, 8 * (last - first + 1), HEADER_SIZE + 8 * first)
            if len(traw) != 8 * (last - first + 1):
                raise CorruptData("container truncated inside the offset table")
            t = np.frombuffer(traw, "<u8")
            base = HEADER_SIZE + 8 * (h["blocks"] + 1)
            _check_span(t, base, size)
            pay = os.pread(fd, int(t[-1] - t[0]), base + int(t[0]))
        finally:
            os.close(fd)
        return head, t, pay
    try:
        import torch
        is_tensor = isinstance(src, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_tensor = False
    if is_tensor:
        src = src.reshape(-1).view(torch.uint8)
        head = src[:HEADER_SIZE].cpu().numpy().tobytes()
        if len(head) < HEADER_SIZE:
            raise CorruptData("container shorter than the 46-byte global header")
        h = _header_fields(head)
        _check_range(h, first, last)
        traw = src[HEADER_SIZE + 8 * first: HEADER_SIZE + 8 * (last + 1)].cpu().numpy().tobytes()
        if len(traw) != 8 * (last - first + 1):
            raise CorruptData("container truncated inside the offset table")
        t = np.frombuffer(traw, "<u8")
        base = HEADER_SIZE + 8 * (h["blocks"] + 1)
        _check_span(t, base, src.numel())
        pay = src[base + int(t[0]): base + int(t[-1])]  # stays on the device
        return head, t, pay
    mv = memoryview(src).cast("B")
    head = bytes(mv[:HEADER_SIZE])
    if len(head) < HEADER_SIZE:
        raise CorruptData("container shorter than the 46-byte global header")
    h = _header_fields(head)
    _check_range(h, first, last)
    traw = bytes(mv[HEADER_SIZE + 8 * first: HEADER_SIZE + 8 * (last + 1)])
    if len(traw) != 8 * (last - first + 1):
        raise CorruptData("container truncated inside the offset table")
    t = np.frombuffer(traw, "<u8")
    base = HEADER_SIZE + 8 * (h["blocks"] + 1)
    _check_span(t, base, mv.nbytes)
    return head, t, mv[base + int(t[0]): base + int(t[-1])]


def _check_range(h, first: int, last: int) -> None:
    if not 0 <= first <= last <= h["blocks"]:
        raise IndexError(f"block range [{first}, {last}) outside the container's {h['blocks']} blocks")


def _check_span(t: np.ndarray, base: int, size: int) -> None:
    if np.any(t[1:] < t[:-1]):
        raise CorruptData("offset table is not nondecreasing")
    if base + int(t[-1]) > size:
        raise CorruptData("payload region shorter than the offset table says")


def decompress_blocks(src, first: int, last: int, device: bool = False):
    """Blocks [first, last) of a container (bytes, CUDA tensor or file path),
    reconstructed on the GPU.  Returns a Dataset (numpy axes, or CUDA tensors
    with ``device=True``); errors name blocks by their index in ``src``."""
    import torch

    from . import _lib
    from .model import Dataset, Precision
    from .pipeline import _check, _decode, _device, parse_header

    head, t, pay = _read_range(src, first, last)
    sub_head = sub_container(head, t, b"", first, last)  # header + rebased table
    if isinstance(pay, torch.Tensor):
        dev = torch.empty(len(sub_head) + pay.numel(), dtype=torch.uint8, device=pay.device)
        dev[: len(sub_head)].copy_(torch.frombuffer(bytearray(sub_head), dtype=torch.uint8))
        dev[len(sub_head):].copy_(pay)
    else:
        dev = torch.frombuffer(bytearray(sub_head + bytes(pay)), dtype=torch.uint8).to(_device())
    h = parse_header(sub_head[:HEADER_SIZE], dev.numel())
    outs, res, _ = _decode(dev, h)
    if res.status != _lib.OK:
        if res.block >= 0:
            res.block += first
        _check(res.status, res)
    n = h.particle_count
    ds = Dataset(axes=tuple(o[:n] for o in outs), precision=Precision(h.precision))
    return ds if device else ds.numpy()


def iter_file_blocks(path, chunk_blocks: int = 4096, device: bool = False):
    """Stream a container file: yields (first_block, Dataset) per chunk of
    ``chunk_blocks`` blocks, reading only that chunk's table and payload."""
    with open(path, "rb") as f:
        head = f.read(HEADER_SIZE)
    if len(head) < HEADER_SIZE:
        raise CorruptData("container shorter than the 46-byte global header")
    blocks = _header_fields(head)["blocks"]
    for first in range(0, blocks, chunk_blocks):
        yield first, decompress_blocks(path, first, min(first + chunk_blocks, blocks), device=device)
