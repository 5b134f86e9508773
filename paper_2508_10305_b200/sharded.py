"""Multi-GPU compression by contiguous, block-aligned particle ranges.

One process per GPU (torchrun / torch.distributed, NCCL on the B200 box).
Blocks are independent, so each rank compresses its own
range with no data-path collective; the only exchanges are scalars
(SURVEY.md §8e):

1. REL mode: all-reduce(MAX) of the two order-preserving range words of
   K1 (encodings of -lo and +hi, model.py:194-195) -> every rank resolves the
   identical global eb_abs, so its blocks are byte-identical to a
   single-GPU run over the concatenated dataset;
2. all-gather of each rank's payload total -> exclusive prefix -> the
   rank's base offset in the global offset table.

Each rank keeps a *local* container (a valid .gpz of its own blocks); the
global file is the global header + entry 0 + every rank's table slice
shifted by its base + every rank's payload, concatenated in rank order
(`to_global_bytes`).  Shards must be block-aligned: every rank except the
last holds a multiple of block_size particles.

The orchestration is written against two hooks (`local_range`,
`local_encode`) so it can be exercised on CPU with the gloo backend in
tests; the product hooks call the CUDA library.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import lib
from .model import CompressConfig, Dataset, EbMode

_I64_MIN = -(1 << 63)


@dataclass
class ShardedContainer:
    local: object            # local container (CUDA uint8 tensor, or bytes in CPU tests)
    rank: int
    world: int
    base: int                # this rank's payload offset in the global payload region
    first_block: int         # global index of this rank's first block
    global_count: int
    global_blocks: int
    local_blocks: int
    header: bytes            # global 46-byte header (every rank knows it)
    global_payload: int = 0  # payload bytes over all ranks (file length - 46 - 8 (B + 1))

    @property
    def local_bytes(self) -> int:
        return int(self.local.numel() if hasattr(self.local, "numel") else len(self.local))


def _allreduce_max_words(words: torch.Tensor) -> None:
    """MAX all-reduce of u64 order-preserving words stored as int64 (in place;
    over NCCL the device words are reduced directly, otherwise via the host)."""
    dev = _comm_device()
    t = words if words.device == dev else words.to(dev)
    t ^= _I64_MIN
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t ^= _I64_MIN
    if t is not words:
        words.copy_(t)


def _gather_ints(v: int, device) -> list[int]:
    t = torch.tensor([v], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [int(x.item()) for x in out]


# ---------------------------------------------------------------- GPU hooks
class _CudaHooks:
    def __init__(self, ds: Dataset, cfg: CompressConfig, timing=None):
        from .pipeline import _check, _device_axes, _stream, _workspace

        self._check, self._stream = _check, _stream
        self.ds, self.cfg, self.timing = ds, cfg, timing
        self.axes = _device_axes(ds)
        self.ptrs = _lib.ptr_array([a.data_ptr() for a in self.axes])
        n, d, p, bs = ds.count, ds.dims, ds.precision.value, cfg.block_size
        wsb = ctypes.c_uint64()
        _check(lib.gpzb_compress_workspace(n, d, p, bs, ctypes.byref(wsb)))
        self.ws = _workspace(wsb.value)
        _check(lib.gpzb_workspace_reset_async(self.ws.data_ptr(), self.ws.numel(), n, bs, _stream()))

    def _ev(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def local_range_words(self) -> torch.Tensor:
        ds, cfg = self.ds, self.cfg
        e0 = self._ev() if self.timing is not None else None
        self._check(lib.gpzb_range_async(self.ptrs, ds.dims, ds.precision.value, ds.count, cfg.block_size,
                                         self.ws.data_ptr(), self.ws.numel(), self._stream()))
        if self.timing is not None:
            self.timing.setdefault("range", []).append((e0, self._ev()))
        return self.ws[40:56].view(torch.int64)  # DevResult.range_w, in place

    def local_encode(self, global_count: int, global_blocks: int):
        """This rank's local container (a valid .gpz of its own blocks),
        allocated at its exact size after the scan; an empty shard gets the
        empty container (header + entry 0)."""
        from .pipeline import _side

        ds, cfg = self.ds, self.cfg
        dev = self.axes[0].device if self.axes else torch.device("cuda", torch.cuda.current_device())
        res = _lib.Result()
        args = (self.ptrs, ds.dims, ds.precision.value, ds.count, float(cfg.error_bound), cfg.eb_mode.value,
                cfg.block_size, cfg.target_segs_per_axis, int(cfg.preserve_order), self.ws.data_ptr(),
                self.ws.numel())
        if ds.count == 0:
            bound = ctypes.c_uint64()
            self._check(lib.gpzb_compress_bound(0, ds.dims, ds.precision.value, cfg.block_size,
                                                cfg.target_segs_per_axis, int(cfg.preserve_order),
                                                ctypes.byref(bound)))
            out = torch.empty(bound.value, dtype=torch.uint8, device=dev)
            st = lib.gpzb_compress(*args, out.data_ptr(), bound.value, self._stream(), ctypes.byref(res))
            return st, res, out[: res.out_len].clone() if st == 0 else None
        nb = (ds.count + cfg.block_size - 1) // cfg.block_size
        rel = cfg.eb_mode is EbMode.RANGE_RELATIVE
        words = self.ws[40:56].view(torch.int64).clone() if rel else None  # the all-reduced range words

        def run(first: bool) -> int:
            if not first:  # a second pass after the side buffer grew (GPZB_NEED_SIDE)
                self._check(lib.gpzb_workspace_reset_async(self.ws.data_ptr(), self.ws.numel(), ds.count,
                                                           cfg.block_size, self._stream()))
            if not first or not rel:  # per-block bounds come from K1 in both modes
                self._check(lib.gpzb_range_async(self.ptrs, ds.dims, ds.precision.value, ds.count, cfg.block_size,
                                                 self.ws.data_ptr(), self.ws.numel(), self._stream()))
            if not first and rel:
                self.ws[40:56].view(torch.int64).copy_(words)
            self._check(lib.gpzb_encode_plan_async(*args, self._stream()))
            side = _side(0)
            self._check(lib.gpzb_encode_async(*args, side.data_ptr(), side.numel(), None, 0, 0, ds.count, nb, 1,
                                              self._stream()))
            return lib.gpzb_compress_result(self.ws.data_ptr(), self.ws.numel(), ds.count, cfg.block_size,
                                            self._stream(), ctypes.byref(res))

        e0 = self._ev() if self.timing is not None else None
        st = run(True)
        if st == _lib.NEED_SIDE:
            _side(0, res.side_bytes)
            st = run(False)
        if st != 0:
            return st, res, None
        out = torch.empty(res.out_len, dtype=torch.uint8, device=dev)
        self._check(lib.gpzb_emit_async(self.ptrs, ds.dims, ds.precision.value, ds.count, float(cfg.error_bound),
                                        cfg.eb_mode.value, cfg.block_size, int(cfg.preserve_order),
                                        self.ws.data_ptr(), self.ws.numel(), _side(0).data_ptr(), out.data_ptr(),
                                        out.numel(), 0, ds.count, nb, 1, self._stream()))
        if e0 is not None:
            self.timing.setdefault("encode", []).append((e0, self._ev()))
        return st, res, out


def _eb_bits(v: float) -> int:
    return struct.unpack("<q", struct.pack("<d", float(v)))[0]


def _global_eb_abs(cfg: CompressConfig, rows: list) -> float:
    """The header's eb_abs: every non-empty rank resolved the same value from
    the all-reduced range words, so take the first one's; a dataset with no
    particles at all keeps the raw bound (pipeline.py:75)."""
    for r in rows:
        if r["count"] > 0:
            return struct.unpack("<d", struct.pack("<q", r["eb_bits"]))[0]
    return float(cfg.error_bound)


def _header(dims, prec, cfg: CompressConfig, eb_abs: float, count: int, blocks: int) -> bytes:
    return struct.pack("<4sHBBBBddIQQ", b"GPZ1", 1, dims, prec, 1 if cfg.preserve_order else 0,
                       cfg.eb_mode.value, float(cfg.error_bound), eb_abs, cfg.block_size, count, blocks)


def compress_device(ds: Dataset, cfg: CompressConfig, *, timing=None, hooks=None) -> ShardedContainer:
    """Compress this rank's block-aligned shard; collective over the default group."""
    rank, world = dist.get_rank(), dist.get_world_size()
    bs = cfg.block_size
    counts = _gather_ints(ds.count, _comm_device())
    for r in range(world - 1):
        if counts[r] % bs:
            raise ValueError(f"rank {r} holds {counts[r]} particles, not a multiple of block_size {bs}")
    g_count = sum(counts)
    first_block = sum((c + bs - 1) // bs for c in counts[:rank])
    g_blocks = sum((c + bs - 1) // bs for c in counts)
    h = hooks if hooks is not None else _CudaHooks(ds, cfg, timing)
    if cfg.eb_mode is EbMode.RANGE_RELATIVE:
        words = h.local_range_words()
        _allreduce_max_words(words)
    st, res, local = h.local_encode(g_count, g_blocks)
    # one all-gather: the first error over ranks in global block order
    # (pipeline.py:80-83; dataset-level errors precede every block error),
    # each rank's payload total (-> its base offset) and its resolved eb_abs
    inf = 1 << 62
    nb = (ds.count + bs - 1) // bs
    key = inf if st == 0 else (-1 if res.block < 0 else first_block + res.block)
    payload = (int(local.numel() if hasattr(local, "numel") else len(local)) - 46 - 8 * (nb + 1)) if st == 0 else 0
    info = torch.tensor([key, st, res.reason, res.axis, payload, _eb_bits(res.eb_abs), ds.count],
                        dtype=torch.int64, device=_comm_device())
    allinfo = [torch.zeros_like(info) for _ in range(world)]
    dist.all_gather(allinfo, info)
    rows = [dict(zip(("key", "st", "reason", "axis", "payload", "eb_bits", "count"), t.tolist())) for t in allinfo]
    win = min(rows, key=lambda r: r["key"])
    if win["key"] != inf:
        from .pipeline import _check

        _check(win["st"], _lib.Result(status=win["st"], reason=win["reason"], block=win["key"], axis=win["axis"]))
    totals = [r["payload"] for r in rows]
    base = sum(totals[:rank])
    header = _header(ds.dims, ds.precision.value, cfg, _global_eb_abs(cfg, rows), g_count, g_blocks)
    return ShardedContainer(local=local, rank=rank, world=world, base=base, first_block=first_block,
                            global_count=g_count, global_blocks=g_blocks, local_blocks=nb, header=header,
                            global_payload=sum(totals))


def compress_batch_device(datasets, cfg: CompressConfig, *, timing=None) -> list:
    """compress_device over several datasets (the fields of one snapshot) with
    one CUDA stream + workspace each, as pipeline.compress_batch_device, and
    ONE collective per exchange for all of them: the shard counts, the range
    words (REL), and the (first error, payload total) records.  Returns one
    ShardedContainer per dataset, each identical to compress_device's."""
    from .pipeline import (_check, _compress_begin, _compress_emit, _compress_encode, _compress_plan, _compress_status,
                           _side_stream)

    rank, world = dist.get_rank(), dist.get_world_size()
    bs = cfg.block_size
    k = len(datasets)
    dev = _comm_device()
    t = torch.tensor([d.count for d in datasets], dtype=torch.int64, device=dev)
    allc = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(allc, t)
    counts = torch.stack(allc).cpu().tolist()  # [rank][dataset]
    for r in range(world - 1):
        for i in range(k):
            if counts[r][i] % bs:
                raise ValueError(f"rank {r} holds {counts[r][i]} particles, not a multiple of block_size {bs}")
    cur = torch.cuda.current_stream()
    start = torch.cuda.Event()
    start.record(cur)
    jobs = []
    for i, ds in enumerate(datasets):
        s = _side_stream(i)
        s.wait_event(start)
        with torch.cuda.stream(s):
            jobs.append(_compress_begin(ds, cfg, i, timing, plan=False))
    if cfg.eb_mode is EbMode.RANGE_RELATIVE:
        live = [j for j in jobs if j.count]
        for i in range(k):
            cur.wait_stream(_side_stream(i))
        if live:
            words = torch.stack([j.ws[40:56].view(torch.int64) for j in live])  # DevResult.range_w of each
            _allreduce_max_words(words)
            for j, w in zip(live, words):
                j.ws[40:56].view(torch.int64).copy_(w)
                j.words = w  # restored if the job encodes again (GPZB_NEED_SIDE)
        for i in range(k):
            _side_stream(i).wait_stream(cur)
    for i, j in enumerate(jobs):
        with torch.cuda.stream(_side_stream(i)):
            _compress_plan(j)
    prev = None  # one encoder at a time, as pipeline.compress_batch_device
    for i, j in enumerate(jobs):
        s = _side_stream(i)
        if prev is not None:
            s.wait_event(prev)
        with torch.cuda.stream(s):
            _compress_encode(j)
            prev = torch.cuda.Event()
            prev.record(s)
    inf = 1 << 62
    rows, locals_ = [], []
    for i, j in enumerate(jobs):
        with torch.cuda.stream(_side_stream(i)):
            st = _compress_status(j)
            if st != 0:
                local = None
            elif j.count == 0:
                local = j.out[: j.res.out_len].clone()  # the empty local container
            else:
                local = _compress_emit(j)
        cur.wait_stream(_side_stream(i))
        first_block = sum((c[i] + bs - 1) // bs for c in counts[:rank])
        key = inf if st == 0 else (-1 if j.res.block < 0 else first_block + j.res.block)
        if local is not None:
            local.record_stream(cur)
        payload = (int(local.numel()) - 46 - 8 * (j.nb + 1)) if local is not None else 0
        rows.append([key, st, j.res.reason, j.res.axis, payload, _eb_bits(j.res.eb_abs), j.count])
        locals_.append(local)
    info = torch.tensor(rows, dtype=torch.int64, device=dev)
    alli = [torch.zeros_like(info) for _ in range(world)]
    dist.all_gather(alli, info)
    alli = torch.stack(alli).cpu().tolist()  # [rank][dataset][5]
    out = []
    for i, (ds, j) in enumerate(zip(datasets, jobs)):
        win = min((alli[r][i] for r in range(world)), key=lambda v: v[0])
        if win[0] != inf:
            key, wst, wreason, waxis = win[:4]
            _check(wst, _lib.Result(status=wst, reason=wreason, block=key, axis=waxis))
        totals = [alli[r][i][4] for r in range(world)]
        g_count = sum(c[i] for c in counts)
        g_blocks = sum((c[i] + bs - 1) // bs for c in counts)
        eb_abs = _global_eb_abs(cfg, [{"count": alli[r][i][6], "eb_bits": alli[r][i][5]} for r in range(world)])
        header = _header(ds.dims, ds.precision.value, cfg, eb_abs, g_count, g_blocks)
        out.append(ShardedContainer(local=locals_[i], rank=rank, world=world, base=sum(totals[:rank]),
                                    first_block=sum((c[i] + bs - 1) // bs for c in counts[:rank]),
                                    global_count=g_count, global_blocks=g_blocks, local_blocks=j.nb,
                                    header=header, global_payload=sum(totals)))
    return out


def decompress_batch_device(scs: list, *, timing=None) -> list:
    """Each rank decodes its own blocks of every container (no exchange)."""
    from .pipeline import decompress_batch_device as dbd

    return dbd([sc.local for sc in scs], timing=timing)


def _comm_device():
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def decompress_device(sc: ShardedContainer, *, timing=None):
    """Each rank decodes its own blocks (no exchange)."""
    from .pipeline import decompress_device as dd

    return dd(sc.local, timing=timing)


def global_pieces(sc: ShardedContainer) -> tuple[int, bytes, int, bytes]:
    """(table offset, table bytes, payload offset, payload bytes) of this rank's
    slice of the global file; rank 0's table slice starts with entry 0."""
    local = sc.local.cpu().numpy().tobytes() if hasattr(sc.local, "cpu") else bytes(sc.local)
    nb = sc.local_blocks
    table = np.frombuffer(local, "<u8", count=nb + 1, offset=46).astype(np.uint64) + np.uint64(sc.base)
    payload = local[46 + 8 * (nb + 1):]
    t_off = 46 + 8 * (sc.first_block + 1)
    p_off = 46 + 8 * (sc.global_blocks + 1) + sc.base
    tbytes = table[1:].astype("<u8").tobytes()
    if sc.rank == 0:
        t_off -= 8
        tbytes = table[:1].astype("<u8").tobytes() + tbytes
    return t_off, tbytes, p_off, payload


def to_global_bytes(sc: ShardedContainer) -> bytes | None:
    """Gather every rank's pieces to rank 0 and return the single-file
    container there (None on other ranks).  Outside any timed region."""
    pieces = global_pieces(sc)
    gathered = [None] * sc.world
    dist.all_gather_object(gathered, pieces)
    if sc.rank != 0:
        return None
    total = max(p_off + len(p) for _, _, p_off, p in gathered)
    buf = bytearray(total)
    buf[:46] = sc.header
    for t_off, t, p_off, p in gathered:
        buf[t_off:t_off + len(t)] = t
        buf[p_off:p_off + len(p)] = p
    return bytes(buf)
