"""Multi-process (world_size 2, gloo, CPU) test of the sharded orchestration:
range all-reduce, error agreement, payload-total all-gather and the global
file assembly.  The per-rank encoder is the oracle here (test-only hooks);
on the GPU box the same orchestration drives the CUDA kernels."""

import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import gpz_oracle as O

MASK = (1 << 64) - 1


def _ukey(v: float) -> int:
    b = struct.unpack("<Q", struct.pack("<d", v))[0]
    k = (~b & MASK) if (b >> 63) else (b | (1 << 63))
    return k - (1 << 64) if k >= (1 << 63) else k


def _ukey_inv(k: int) -> float:
    k &= MASK
    b = (k & 0x7FFFFFFFFFFFFFFF) if (k >> 63) else (~k & MASK)
    return struct.unpack("<d", struct.pack("<Q", b))[0]


class OracleHooks:
    """Stand-in for the CUDA hooks: same contract, oracle arithmetic."""

    def __init__(self, axes, cfg):
        self.axes, self.cfg = axes, cfg

    def local_range_words(self):
        if self.axes[0].size == 0:  # an empty shard: the zeroed words (below every key)
            self.words = torch.zeros(2, dtype=torch.int64)
            return self.words
        lo = min(float(a.min()) for a in self.axes)
        hi = max(float(a.max()) for a in self.axes)
        self.words = torch.tensor([_ukey(-lo), _ukey(hi)], dtype=torch.int64)
        return self.words

    def local_encode(self, g_count, g_blocks):
        import paper_2508_10305_b200._lib as L

        c = self.cfg
        if self.axes[0].size == 0:
            blob = O.assemble(len(self.axes), O.F32, O.Config(c.error_bound, c.eb_mode.value, c.block_size), 0.0,
                              0, [])
            return 0, L.Result(status=0, eb_abs=0.0), blob
        if c.eb_mode.value == O.RANGE_RELATIVE:
            lo, hi = -_ukey_inv(int(self.words[0])), _ukey_inv(int(self.words[1]))
            span = hi - lo
            eb_abs = c.error_bound * (span if span > 0 else 1.0)
        else:
            eb_abs = c.error_bound
        oc = O.Config(c.error_bound, c.eb_mode.value, c.block_size, c.target_segs_per_axis, c.preserve_order)
        n = self.axes[0].size
        pay = []
        for i, s in enumerate(range(0, n, c.block_size)):
            try:
                pay.append(O.encode_block([a[s:s + c.block_size] for a in self.axes], eb_abs, oc, O.F32))
            except O.OracleError as exc:
                st = L.WIDTH if isinstance(exc, O.WidthOverflow) else L.DOMAIN
                return st, L.Result(status=st, reason=3, block=i, axis=0), None
        n_blk = len(pay)
        blob = O.assemble(len(self.axes), O.F32, oc, eb_abs, n, pay)
        assert n_blk == (n + c.block_size - 1) // c.block_size
        return 0, L.Result(status=0, eb_abs=eb_abs), blob


def _run(rank, world, port, case, q, path=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2508_10305_b200 as gz
        from paper_2508_10305_b200 import sharded

        full = O.gen_clusters(5000, dims=3, seed=11)
        if case == "overflow":
            full[0] = full[0].astype(np.float32)
            full[0][3500] = 3e38  # block 3 (rank 1's first block) overflows in ABS mode
        cuts = [0, 0, 5000] if case == "empty" else [0, 3072, 5000]  # "empty": rank 0 holds no particles
        local = [a[cuts[rank]:cuts[rank + 1]] for a in full]
        mode = gz.EbMode.ABSOLUTE if case == "overflow" else gz.EbMode.RANGE_RELATIVE
        cfg = gz.CompressConfig(error_bound=1e-3 if case != "overflow" else 1e-6, eb_mode=mode)
        ds = gz.Dataset.from_axes(local)
        try:
            sc = sharded.compress_device(ds, cfg, hooks=OracleHooks(local, cfg))
        except gz.GpzError as exc:
            q.put((rank, "err", type(exc).__name__, str(exc)))
            return
        if case == "file":
            from paper_2508_10305_b200 import gpzfile

            gpzfile.write_sharded(path, sc)
            if rank == 0:
                with open(path, "rb") as f:
                    got = f.read()
                want = O.compress(full, O.Config(cfg.error_bound, mode.value))
                q.put((rank, "ok", got == want, len(want)))
            else:
                q.put((rank, "ok", True, 0))
            return
        blob = sharded.to_global_bytes(sc)
        if rank == 0:
            want = O.compress(full, O.Config(cfg.error_bound, mode.value))
            q.put((rank, "ok", blob == want, len(want)))
        else:
            q.put((rank, "ok", True, 0))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case", ["rel", "overflow", "file", "empty"])
def test_sharded_global_container_equals_single_process(case, tmp_path):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    path = str(tmp_path / "sharded.gpz")
    procs = [ctx.Process(target=_run, args=(r, 2, port, case, q, path)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    out.sort()
    if case in ("rel", "file", "empty"):
        assert out[0][1:3] == ("ok", True), out
        assert out[1][1] == "ok"
    else:
        # both ranks raise the same first error, with the global block index
        for r in out:
            assert r[1] == "err" and r[2] == "WidthOverflow" and r[3].startswith("block 3"), out


def _run_cuda(rank, world, port, q, path):
    """Both ranks on cuda:0 (gloo for the scalar exchanges): the product CUDA
    hooks of sharded.compress_device, exactly as under torchrun with NCCL."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2508_10305_b200 as gz
        from paper_2508_10305_b200 import gpzfile, sharded

        full = O.gen_clusters(400_000, dims=3, seed=21)
        cut = 196 * 1024
        sl = slice(0, cut) if rank == 0 else slice(cut, None)
        ds = gz.Dataset.from_axes([torch.from_numpy(a[sl].copy()).cuda() for a in full])
        cfg = gz.CompressConfig(error_bound=1e-3)
        sc = sharded.compress_device(ds, cfg)
        blob = sharded.to_global_bytes(sc)
        gpzfile.write_sharded(path, sc)
        rec = sharded.decompress_device(sc)
        if rank == 0:
            want = gz.compress(gz.Dataset.from_axes(full), cfg)
            with open(path, "rb") as f:
                disk = f.read()
            full_rec = gz.decompress(want)
            ok_rec = all(np.array_equal(r.cpu().numpy(), w[:cut]) for r, w in zip(rec.axes, full_rec.axes))
            q.put((rank, blob == want, disk == want, ok_rec))
        else:
            full_rec = gz.decompress(gz.compress(gz.Dataset.from_axes(full), cfg))
            ok_rec = all(np.array_equal(r.cpu().numpy(), w[cut:]) for r, w in zip(rec.axes, full_rec.axes))
            q.put((rank, True, True, ok_rec))
        # an empty shard on rank 0: its local container is the valid empty
        # one and the global header carries rank 1's eb_abs
        sl = slice(0, 0) if rank == 0 else slice(0, None)
        ds = gz.Dataset.from_axes([torch.from_numpy(a[sl].copy()).cuda() for a in full])
        sc = sharded.compress_device(ds, cfg)
        blob = sharded.to_global_bytes(sc)
        assert gz.decompress_device(sc.local).count == ds.count
        if rank == 0:
            q.put((rank + 10, blob == want, True, True))
        else:
            q.put((rank + 10, True, True, True))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_cuda_hooks_two_ranks_one_gpu(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    path = str(tmp_path / "sharded_cuda.gpz")
    procs = [ctx.Process(target=_run_cuda, args=(r, 2, port, q, path)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(2 * len(procs)))
    for p in procs:
        p.join(timeout=60)
    assert out == [(0, True, True, True), (1, True, True, True), (10, True, True, True), (11, True, True, True)], out


def _run_cuda_batch(rank, world, port, q):
    """sharded.compress_batch_device over two fields (one stream each, one
    collective per exchange): every container equals the single-process one."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2508_10305_b200 as gz
        from paper_2508_10305_b200 import sharded

        rng = np.random.default_rng(5)
        pos = O.gen_clusters(300_000, dims=3, seed=22)
        vel = [(rng.normal(0, 0.3, 300_000) + rng.normal(0, 0.05, 300_000)).astype(np.float32) for _ in range(3)]
        cut = 150 * 1024
        sl = slice(0, cut) if rank == 0 else slice(cut, None)
        shards = [gz.Dataset.from_axes([torch.from_numpy(a[sl].copy()).cuda() for a in f]) for f in (pos, vel)]
        ok = []
        for mode in (gz.EbMode.RANGE_RELATIVE, gz.EbMode.ABSOLUTE):
            cfg = gz.CompressConfig(error_bound=1e-3, eb_mode=mode)
            scs = sharded.compress_batch_device(shards, cfg)
            blobs = [sharded.to_global_bytes(sc) for sc in scs]
            recs = sharded.decompress_batch_device(scs)
            for f, blob, rec in zip((pos, vel), blobs, recs):
                want = gz.compress(gz.Dataset.from_axes(f), cfg)
                full_rec = gz.decompress(want)
                ok.append(all(np.array_equal(r.cpu().numpy(), w[sl]) for r, w in zip(rec.axes, full_rec.axes)))
                if rank == 0:
                    ok.append(blob == want)
        # an overflowing block on rank 1 (second field): every rank raises the
        # single-process error, global block index included
        bad = [a.copy() for a in vel]
        bad[1][cut + 5000] = 3e38
        cfg = gz.CompressConfig(error_bound=1e-6, eb_mode=gz.EbMode.ABSOLUTE)
        shards[1] = gz.Dataset.from_axes([torch.from_numpy(a[sl].copy()).cuda() for a in bad])
        try:
            gz.compress(gz.Dataset.from_axes(bad), cfg)
            want_err = None
        except gz.GpzError as exc:
            want_err = (type(exc).__name__, str(exc))
        try:
            sharded.compress_batch_device(shards, cfg)
            got_err = None
        except gz.GpzError as exc:
            got_err = (type(exc).__name__, str(exc))
        ok.append(want_err is not None and got_err == want_err)
        q.put((rank, all(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_batch_two_ranks_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_cuda_batch, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert out == [(0, True), (1, True)], out
