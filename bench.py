#!/usr/bin/env python
"""GPZ B200 compress / decompress throughput (BASELINE.json configs).

Workloads (--workload; synthetic data generated on the GPU, no network):

* hacc280m (default, configs[1]): per GPU, 280M particles
  x 6 float32 fields stored as two dims=3 datasets (positions xyz,
  velocities vxvyvz), each compressed with its own range-relative bound 1e-3,
  block_size 1024, target 32.  8192 Gaussian clusters stored cluster by
  cluster; positions sigma 0.002 in the unit box, velocities = per-cluster
  bulk N(0, 0.3) + per-particle N(0, 0.05).  Weak scaling.
* lidar500m (configs[2], C3): per GPU, a 500M-point xyz float32 scan-line
  terrain cloud, rel-eb 1e-4.  Weak scaling.
* decomp1b (configs[3], C4): per GPU, 1B clustered xyz float32 particles
  compressed (untimed) at rel-eb 1e-2 / 1e-3 / 1e-4; a step decompresses the
  three containers and `value` is decompress GB/s.  Weak scaling.
* snapshot2b (configs[4], C5): ONE 2B-particle 6-field snapshot (hacc family)
  split by block-aligned particle range over the N ranks.  Strong scaling.

A step = compress every dataset, then decompress every container (decomp1b:
decompress only).  `value` is compress GB/s (decomp1b: decompress GB/s):
input bytes of all ranks / the max over ranks of the device time of the
compress calls (inputs resident in HBM).  Inputs exceed the 126 MB L2 by
> 40x, so no flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gpzb|reference] [--workload W]

--gpus N > 1 without torchrun in the environment re-launches itself under
torch.distributed.run with N ranks (NCCL, NCCL_DEBUG=INFO for the
communicator lines).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress/decompress GB/s at rel-eb 1e-3 on 1/2/4/8 B200; compression ratio"
PARTICLES = 280_000_000
CLUSTERS = 8192
CPU_SAMPLE = 8 * 1024 * 1024  # particles per dataset for the CPU baseline (8192 blocks)
CPU_SAMPLE_1 = 1024 * 1024    # particles per dataset for the single-worker CPU figure
WORKLOADS = {
    "hacc280m": {"config": 1, "desc": "HACC-like 280M particles x 6 float32 fields (x,y,z,vx,vy,vz) per GPU, "
                                      "two dims=3 datasets, rel-eb 1e-3, block 1024, target 32",
                 "particles": PARTICLES, "scaling": "weak"},
    "lidar500m": {"config": 2, "desc": "LiDAR-style clustered point cloud 500M points xyz float32 per GPU, "
                                       "rel-eb 1e-4, block 1024, target 32",
                  "particles": 500_000_000, "scaling": "weak"},
    "decomp1b": {"config": 3, "desc": "decompression sweep over rel-eb 1e-2/1e-3/1e-4 on 1B clustered xyz "
                                      "float32 particles per GPU", "particles": 1_000_000_000, "scaling": "weak"},
    "snapshot2b": {"config": 4, "desc": "2B-particle 6-field snapshot (hacc family, two dims=3 datasets, rel-eb "
                                        "1e-3) sharded by block-aligned particle range across the ranks",
                   "particles": 2_000_000_000, "scaling": "strong"},
}


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["gpzb", "reference"], default="gpzb")
    p.add_argument("--workload", choices=sorted(WORKLOADS), default="hacc280m")
    p.add_argument("--particles", type=int, default=None,
                   help="particles per GPU per dataset (snapshot2b: in total); default: the workload's")
    p.add_argument("--cpu-sample", type=int, default=CPU_SAMPLE)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--compress-only", action="store_true", help="experiments: skip decompress")
    p.add_argument("--per-call", action="store_true",
                   help="one compress_device / decompress_device call per field instead of the batched calls")
    a = p.parse_args()
    if a.particles is None:
        a.particles = WORKLOADS[a.workload]["particles"]
    return a


def _relaunch_distributed(args) -> None:
    """`python bench.py --gpus N` outside torchrun: run N ranks under
    torch.distributed.run (one process per GPU) and exit with its status."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


# ------------------------------------------------------------------ workload
def gen_hacc(n: int, seed: int, device) -> tuple[list, list]:
    """Positions and velocities, cluster-contiguous (bench._gaussian_clusters family)."""
    g = torch.Generator(device=device).manual_seed(seed)
    centers = torch.rand(CLUSTERS, 3, generator=g, device=device, dtype=torch.float64)
    bulk = 0.3 * torch.randn(CLUSTERS, 3, generator=g, device=device, dtype=torch.float64)
    assign = (torch.arange(n, device=device, dtype=torch.int64) * CLUSTERS) // n
    pos, vel = [], []
    for a in range(3):
        pos.append((centers[assign, a] + 0.002 * torch.randn(n, generator=g, device=device,
                                                              dtype=torch.float64)).float())
    for a in range(3):
        vel.append((bulk[assign, a] + 0.05 * torch.randn(n, generator=g, device=device,
                                                          dtype=torch.float64)).float())
    del assign
    return pos, vel


def gen_lidar(n: int, seed: int, device):
    """configs[2]: 2.5-D terrain in scan-line order — jittered x/y lattice
    rows, z a smooth height field plus sensor noise."""
    g = torch.Generator(device=device).manual_seed(seed)
    w = int(np.ceil(np.sqrt(n)))
    i = torch.arange(n, device=device, dtype=torch.int64)
    f64 = torch.float64
    x = (i % w).to(f64) * 0.05 + (torch.rand(n, generator=g, device=device, dtype=f64) * 2 - 1) * 0.01
    y = (i // w).to(f64) * 0.05 + (torch.rand(n, generator=g, device=device, dtype=f64) * 2 - 1) * 0.01
    del i
    z = 10.0 * torch.sin(x / 50.0) * torch.cos(y / 37.0) + 0.002 * torch.randn(n, generator=g, device=device,
                                                                                  dtype=f64)
    return [x.float(), y.float(), z.float()]


def gen_clusters(n: int, clusters: int, sigma: float, seed: int, device):
    """configs[3]: cluster-contiguous Gaussian clusters in the unit box."""
    g = torch.Generator(device=device).manual_seed(seed)
    centers = torch.rand(clusters, 3, generator=g, device=device, dtype=torch.float64)
    out = []
    for a in range(3):
        assign = (torch.arange(n, device=device, dtype=torch.int64) * clusters) // n
        v = centers[assign, a] + sigma * torch.randn(n, generator=g, device=device, dtype=torch.float64)
        del assign
        out.append(v.float())
    return out


SHARD_CHUNK = 1 << 26


def gen_snapshot_shard(total: int, lo: int, hi: int, seed: int, device):
    """configs[4]: particles [lo, hi) of ONE `total`-particle snapshot of the
    hacc family.  Cluster centres and bulk velocities come from `seed`; the
    noise of each 2^26-particle chunk from (seed, chunk), so every rank count
    N sees the same global dataset.  Returns (pos, vel) float32 axes."""
    g = torch.Generator(device=device).manual_seed(seed)
    centers = torch.rand(CLUSTERS, 3, generator=g, device=device, dtype=torch.float64)
    bulk = 0.3 * torch.randn(CLUSTERS, 3, generator=g, device=device, dtype=torch.float64)
    n = hi - lo
    pos = [torch.empty(n, device=device, dtype=torch.float32) for _ in range(3)]
    vel = [torch.empty(n, device=device, dtype=torch.float32) for _ in range(3)]
    for c in range(lo // SHARD_CHUNK, (hi + SHARD_CHUNK - 1) // SHARD_CHUNK):
        c0, c1 = c * SHARD_CHUNK, min((c + 1) * SHARD_CHUNK, total)
        gc = torch.Generator(device=device).manual_seed(seed * 1_000_003 + c)
        assign = (torch.arange(c0, c1, device=device, dtype=torch.int64) * CLUSTERS) // total
        noise = [torch.randn(c1 - c0, generator=gc, device=device, dtype=torch.float64) for _ in range(6)]
        a0, a1 = max(c0, lo), min(c1, hi)
        if a0 >= a1:
            continue
        src = slice(a0 - c0, a1 - c0)
        dst = slice(a0 - lo, a1 - lo)
        for a in range(3):
            pos[a][dst] = (centers[assign[src], a] + 0.002 * noise[a][src]).float()
            vel[a][dst] = (bulk[assign[src], a] + 0.05 * noise[3 + a][src]).float()
        del assign, noise
    return pos, vel


def checksum(axes) -> str:
    s = 0
    for a in axes:
        s = (s * 1000003 + int(a.view(torch.int32).to(torch.int64).sum().item())) & 0xFFFFFFFFFFFF
    return f"{s:012x}"


# ------------------------------------------------------------------ clocks
class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region: NVML in
    a sampling thread (every 5 ms, so short regions still get samples), else
    an `nvidia-smi -lms 50` subprocess."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.summary = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
            self.bits = [getattr(pynvml, "nvmlClocksThrottleReason" + n, d) for n, d in
                         (("HwSlowdown", 0x8), ("HwThermalSlowdown", 0x40), ("SwThermalSlowdown", 0x20),
                          ("SwPowerCap", 0x4))]
            self.nvml = pynvml
        except Exception:  # noqa: BLE001 - no NVML: fall back to nvidia-smi
            self.nvml = None

    def _sample(self):
        import time as _t

        nv = self.nvml
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.handle)
                for nm, b in zip(self.NAMES, self.bits):
                    if r & b:
                        self.reasons.add(nm)
            except Exception:  # noqa: BLE001
                return
            _t.sleep(0.005)

    def __enter__(self):
        if self.nvml is not None:
            import threading

            self.sm, self.reasons = [], set()
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._sample, daemon=True)
            self.thread.start()
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=5)
            sm = self.sm
            self.summary = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_sm or None,
                            "samples": len(sm), "reasons": sorted(self.reasons), "source": "nvml"}
            return
        if self.proc is None:
            self.summary = None
            return
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], 0.0, set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        self.summary = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                        "samples": len(sm), "reasons": sorted(reasons), "source": "nvidia-smi"}


# ------------------------------------------------------------------ CPU side
def _cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def _enc_chunk(args):
    from oracle import gpz_oracle as O

    axes, eb, eb_abs, bs = args
    return [O.encode_block([a[s:s + bs] for a in axes], eb_abs, O.Config(eb, block_size=bs), O.F32)
            for s in range(0, axes[0].size, bs)]


def _dec_chunk(args):
    from oracle import gpz_oracle as O

    payloads, h = args
    return [O.decode_block(p, h) for p in payloads]


def cpu_oracle_round(samples, cores, pool):
    """The reference's algorithm on the host (oracle/gpz_oracle.py, a
    restatement of /root/reference/pkg/src/gpz; pipeline.py:85-89 maps
    blocks over `workers` processes the same way): compress + decompress of
    each (axes, rel-eb) sample, blocks split over `cores` processes (pool
    None: in this process).  Returns (compress_s, decompress_s, bytes)."""
    from oracle import gpz_oracle as O

    bs = 1024
    t_c = t_d = 0.0
    nbytes = 0
    for axes, eb in samples:
        n = axes[0].size
        nb = (n + bs - 1) // bs
        per = (nb + cores - 1) // cores
        t0 = time.perf_counter()
        eb_abs = O.absolute_bound(axes, O.Config(eb))
        jobs = [([a[i * per * bs:(i + 1) * per * bs] for a in axes], eb, eb_abs, bs) for i in range(cores)
                if i * per * bs < n]
        parts = pool.map(_enc_chunk, jobs) if pool is not None else [_enc_chunk(j) for j in jobs]
        payloads = [p for part in parts for p in part]
        blob = O.assemble(3, O.F32, O.Config(eb), eb_abs, n, payloads)
        t1 = time.perf_counter()
        h, table, pay = O.read_container(blob)
        jobs = [([pay[int(table[j]):int(table[j + 1])] for j in range(i * per, min((i + 1) * per, nb))], h)
                for i in range(cores) if i * per < nb]
        parts = pool.map(_dec_chunk, jobs) if pool is not None else [_dec_chunk(j) for j in jobs]
        _ = [np.concatenate([b[a] for part in parts for b in part]) for a in range(3)]
        t2 = time.perf_counter()
        t_c += t1 - t0
        t_d += t2 - t1
        nbytes += n * 3 * 4
    return t_c, t_d, nbytes


def make_pool(cores):
    import multiprocessing as mp

    return mp.get_context("fork").Pool(cores)


# ------------------------------------------------------------------ workloads
class Job:
    """One dataset + config of the workload (decomp1b: one per bound)."""

    def __init__(self, name, ds, cfg):
        self.name, self.ds, self.cfg = name, ds, cfg


def shard_range(total: int, world: int, rank: int, bs: int = 1024) -> tuple[int, int]:
    """Block-aligned contiguous particle range of `rank` (sharded.py contract:
    every rank but the last holds whole blocks)."""
    per = ((total + bs - 1) // bs) // world  # whole blocks per rank; the last rank takes the rest
    lo = rank * per * bs
    return lo, (total if rank == world - 1 else lo + per * bs)


def build_jobs(args, world, rank, dev, gz):
    wl = args.workload
    n = args.particles
    if wl in ("hacc280m", "lidar500m", "decomp1b") and world > 1 and rank < world - 1:
        n = (n + 1023) // 1024 * 1024  # sharded path: whole blocks on every rank but the last
    if wl == "hacc280m":
        pos, vel = gen_hacc(n, 280 + 1000 * rank, dev)
        cfg = gz.CompressConfig(error_bound=1e-3)
        return [Job("pos", gz.Dataset.from_axes(pos), cfg), Job("vel", gz.Dataset.from_axes(vel), cfg)], n
    if wl == "lidar500m":
        ax = gen_lidar(n, 500 + 1000 * rank, dev)
        return [Job("lidar", gz.Dataset.from_axes(ax), gz.CompressConfig(error_bound=1e-4))], n
    if wl == "decomp1b":
        ds = gz.Dataset.from_axes(gen_clusters(n, 32768, 0.002, 1000 + 1000 * rank, dev))
        return [Job(f"eb{eb:g}", ds, gz.CompressConfig(error_bound=eb)) for eb in (1e-2, 1e-3, 1e-4)], n
    lo, hi = shard_range(n, world, rank)
    pos, vel = gen_snapshot_shard(n, lo, hi, 2000, dev)
    cfg = gz.CompressConfig(error_bound=1e-3)
    return [Job("pos", gz.Dataset.from_axes(pos), cfg), Job("vel", gz.Dataset.from_axes(vel), cfg)], hi - lo


def _load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ------------------------------------------------------------------ main
def main():
    args = parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return _relaunch_distributed(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    share = os.environ.get("GPZB_BENCH_SHARE_GPU") == "1"
    if world > 1 and not share and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        return run_reference(args, world, rank)

    # GPZB_BENCH_SHARE_GPU=1: every rank on cuda:0 over gloo (exercises the
    # sharded path on a one-GPU box; never used for reported numbers)
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines: nranks, NVLS / P2P transports
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
    import paper_2508_10305_b200 as gz
    from paper_2508_10305_b200 import sharded

    wl = WORKLOADS[args.workload]
    jobs, n_local = build_jobs(args, world, rank, dev, gz)
    decomp_only = args.workload == "decomp1b"
    in_bytes = sum(j.ds.nbytes for j in jobs)  # bytes this rank compresses (decomp1b: decompresses) per step
    by_cfg: dict = {}
    for j in jobs:
        by_cfg.setdefault(id(j.cfg), []).append(j)
    groups = list(by_cfg.values())

    def compress_all(timing=None):
        conts = []
        for grp in groups:
            if args.per_call:
                for j in grp:
                    conts.append(sharded.compress_device(j.ds, j.cfg, timing=timing) if world > 1
                                 else gz.compress_device(j.ds, j.cfg, timing=timing))
            elif world > 1:
                conts += sharded.compress_batch_device([j.ds for j in grp], grp[0].cfg, timing=timing)
            else:
                conts += gz.compress_batch_device([j.ds for j in grp], grp[0].cfg, timing=timing)
        return conts

    def decompress_all(conts, timing=None):
        if args.per_call:
            return [(sharded.decompress_device(c, timing=timing) if world > 1
                     else gz.decompress_device(c, timing=timing)) for c in conts]
        if world > 1:
            return sharded.decompress_batch_device(conts, timing=timing)
        return gz.decompress_batch_device(conts, timing=timing)

    def csize(c):
        return c.local_bytes if world > 1 else c.numel()

    fixed = compress_all() if decomp_only else None  # decomp1b: containers made once, outside the timing

    def one_step(timing=None):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        c = torch.cuda.Event(enable_timing=True)
        a.record()
        conts = fixed if decomp_only else compress_all(timing)
        b.record()
        recs = None if args.compress_only else decompress_all(conts, timing)
        c.record()
        torch.cuda.synchronize()
        sizes = [csize(x) for x in conts]
        del conts, recs
        return a.elapsed_time(b) / 1e3, b.elapsed_time(c) / 1e3, sizes

    for _ in range(args.warmup):
        one_step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    timing: dict = {}
    tcs, tds = [], []
    from paper_2508_10305_b200._lib import lib as _gl

    launches0 = _gl.gpzb_kernel_launches()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            tc, td, sizes = one_step(timing)
            tcs.append(tc)
            tds.append(td)
    torch.cuda.synchronize()
    launches = int(_gl.gpzb_kernel_launches() - launches0)
    if world > 1:
        torch.distributed.barrier()
    t_c, t_d = sum(tcs), sum(tds)
    cont_local = float(sum(sizes))
    if world > 1:
        import torch.distributed as dist

        cdev = "cpu" if share else dev
        t = torch.tensor([t_c, t_d], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_c, t_d = t.tolist()
        z = torch.tensor([cont_local, float(in_bytes)], dtype=torch.float64, device=cdev)
        dist.all_reduce(z)
        total_container, job_bytes = z.tolist()
    else:
        total_container, job_bytes = cont_local, float(in_bytes)
    steps = args.steps
    comp_gbps = job_bytes * steps / t_c / 1e9 if not decomp_only else None
    decomp_gbps = job_bytes * steps / t_d / 1e9 if t_d > 0 else None
    cr = job_bytes / total_container

    peaks = _load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = ("MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)" if "hbm_gbs" in peaks
                else "B200_PROFILING.md fallback")

    # ---- per-call kernel durations (one job at a time, after the timed region)
    per_job = {}
    for j in jobs:
        t: dict = {}
        for _ in range(2):
            cc = gz.compress_device(j.ds, j.cfg, timing=t)
            if not args.compress_only:
                rr = gz.decompress_device(cc, timing=t)
                del rr
            size = cc.numel()
            del cc
        torch.cuda.synchronize()
        last = {k: v[-1][0].elapsed_time(v[-1][1]) for k, v in t.items()}
        per_job[j.name] = {"input_bytes": j.ds.nbytes, "container_bytes": size, "cr": j.ds.nbytes / size,
                           "range_ms": last.get("range"), "encode_ms": last.get("encode"),
                           "decode_ms": last.get("decode")}
    traffic_db = _load_json(os.path.join(ROOT, "profiles", "traffic.json")).get(args.workload, {})
    # the dominant kernel: the slowest encode call (decomp1b: decode call)
    kind = "decode" if decomp_only else "encode"
    dom = max(per_job, key=lambda k: per_job[k][f"{kind}_ms"] or 0.0)
    pj = per_job[dom]
    alg = pj["input_bytes"] + pj["container_bytes"]  # read N*d*s + write C (encode) / read C + write N*d*s (decode)
    tr = traffic_db.get(dom, {}).get(f"{kind}_call_dram_bytes")
    roof = {"bound": "hbm",
            "kernel": (f"{dom} {kind} call: " + ("k_encode_small / k_encode_warp / k_encode (K2) + k_scan_sizes (K3a) "
                                                 "+ k_copy_payloads (K3b)" if kind == "encode" else
                                                 "k_decode_plan (K4a) + k_decode_warp (K4w) + k_decode_list (K4)")),
            "achieved": alg / (pj[f"{kind}_ms"] / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": alg / (pj[f"{kind}_ms"] / 1e3) / 1e9 / hbm, "traffic": tr,
            "traffic_over_algorithmic": (tr / alg) if tr else None,
            "algorithmic_bytes_per_launch": alg, "avg_launch_ms": pj[f"{kind}_ms"], "peak_source": peak_src,
            "timing": "CUDA events on the launching stream around one call, after the timed region",
            "traffic_source": "profiles/traffic.json (ncu dram__bytes_read.sum + dram__bytes_write.sum summed "
                              "over the call's kernels)" if tr else None}
    step_roof = {"decompress_frac": (in_bytes + cont_local) * steps / t_d / 1e9 / hbm if t_d > 0 else None}
    if not decomp_only:
        step_roof["compress_frac"] = (2 * in_bytes + cont_local) * steps / t_c / 1e9 / hbm
    step_roof["note"] = ("per rank: compress A_c = 2*N*d*s + C (REL: the range pass is a mandatory read), "
                         "decompress A_d = C + N*d*s, over the device time of the step's calls")

    value = comp_gbps if not decomp_only else decomp_gbps
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": (t_c if not decomp_only else t_d) / steps * 1e3,
        "higher_is_better": True,
        "scaling": wl["scaling"],
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (GPU-generated, fixed seeds; no network)",
        "config": {"workload": f"{args.workload}: {wl['desc']}", "baseline_config": wl["config"],
                   "value_is": "decompress GB/s" if decomp_only else "compress GB/s",
                   "particles_per_gpu": n_local, "datasets": [j.name for j in jobs],
                   "input_bytes_per_gpu": in_bytes,
                   "l2": f"inputs {in_bytes / 1e9:.2f} GB per GPU >> 126 MB L2, no flush needed",
                   "input_checksum_rank0": checksum([a for j in jobs[:2] for a in j.ds.axes])},
        "compression_ratio": cr,
        "decompress": {"value": decomp_gbps, "unit": "GB/s", "ms_per_step": t_d / steps * 1e3},
        "roofline": roof,
        "step_roofline": step_roof,
        "per_job": per_job,
        "gpu_launches": launches,
        "clocks": clk.summary,
    }
    if decomp_only:
        line["compress_untimed_note"] = "containers compressed once before the timed region"
    if rank == 0 and not args.no_e2e and args.workload != "snapshot2b":
        line["e2e"] = e2e_numbers(gz, jobs, args, decomp_only)
        if "decompress" in line["e2e"]:
            line["decompress"]["e2e"] = line["e2e"].pop("decompress")
    elif args.workload == "snapshot2b":
        line["e2e_note"] = "not measured for the strong-scaling snapshot (48 GB of pinned host buffers)"
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(jobs, args.cpu_sample)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def e2e_numbers(gz, jobs, args, decomp_only):
    """The same metric through the public API from pinned HOST buffers:
    H2D of the inputs, compress, D2H of the container to Python bytes; then
    decompress(bytes) -> numpy (H2D container, decode, D2H of the axes)."""
    hosts = {}
    for j in jobs:
        if id(j.ds) not in hosts:
            hosts[id(j.ds)] = gz.Dataset.from_axes([a.cpu().pin_memory() for a in j.ds.axes])
    torch.cuda.synchronize()
    blobs = [gz.compress(hosts[id(j.ds)], j.cfg) for j in jobs]  # warm-up
    for b in blobs:
        gz.decompress(b)
    tc = td = 0.0
    reps = max(1, min(args.steps, 3 if not decomp_only else 1))
    cbytes = 0
    in_bytes = sum(j.ds.nbytes for j in jobs)
    for _ in range(reps):
        for j, b in zip(jobs, blobs):
            t0 = time.perf_counter()
            blob = gz.compress(hosts[id(j.ds)], j.cfg) if not decomp_only else b
            t1 = time.perf_counter()
            gz.decompress(blob)
            t2 = time.perf_counter()
            tc += t1 - t0
            td += t2 - t1
            cbytes += len(blob)
    dec = {"value": in_bytes * reps / td / 1e9, "unit": "GB/s", "h2d_bytes_per_step": cbytes // reps,
           "d2h_bytes_per_step": in_bytes, "api": "paper_2508_10305_b200.decompress(bytes) -> numpy Dataset"}
    if decomp_only:
        return dict(dec, reps=reps)
    return {"value": in_bytes * reps / tc / 1e9, "unit": "GB/s", "h2d_bytes_per_step": in_bytes,
            "d2h_bytes_per_step": cbytes // reps, "reps": reps,
            "api": "paper_2508_10305_b200.compress(Dataset of pinned CPU tensors) -> bytes", "decompress": dec}


def cpu_baseline(jobs, sample):
    """The reference algorithm on this box's host cores, on the first
    `sample` particles of each job (all cores), and on the first
    CPU_SAMPLE_1 particles with one worker (the reference's workers=1)."""
    samples = [([a[:sample].cpu().numpy() for a in j.ds.axes], j.cfg.error_bound) for j in jobs]
    cores = _cpu_cores()
    with make_pool(cores) as pool:
        t_c, t_d, nbytes = cpu_oracle_round(samples, cores, pool)
    s1 = [([a[:CPU_SAMPLE_1] for a in ax], eb) for ax, eb in samples]
    c1, d1, b1 = cpu_oracle_round(s1, 1, None)
    return {"value": nbytes / t_c / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
            "decompress_value": nbytes / t_d / 1e9, "cpu_model": _cpu_model(),
            "sample": f"first {sample} particles of each of the {len(jobs)} jobs ({nbytes} bytes), "
                      f"oracle/gpz_oracle.py per-block encode/decode spread over {cores} processes",
            "workers_1": {"value": b1 / c1 / 1e9, "decompress_value": b1 / d1 / 1e9, "cores": 1,
                          "sample": f"first {CPU_SAMPLE_1} particles of each job, one process"}}


def reference_sample(args):
    """A bounded CPU sample of the workload (same generator family, CPU
    generator): [(axes, rel-eb)]."""
    n = args.cpu_sample
    cpu = torch.device("cpu")
    wl = args.workload
    if wl in ("hacc280m", "snapshot2b"):
        import math

        k = max(1, int(math.ceil(CLUSTERS * n / args.particles)))
        g = torch.Generator().manual_seed(280)
        centers = torch.rand(k, 3, generator=g, dtype=torch.float64)
        bulk = 0.3 * torch.randn(k, 3, generator=g, dtype=torch.float64)
        assign = (torch.arange(n, dtype=torch.int64) * k) // n
        pos = [(centers[assign, a] + 0.002 * torch.randn(n, generator=g, dtype=torch.float64)).float().numpy()
               for a in range(3)]
        vel = [(bulk[assign, a] + 0.05 * torch.randn(n, generator=g, dtype=torch.float64)).float().numpy()
               for a in range(3)]
        return [(pos, 1e-3), (vel, 1e-3)]
    if wl == "lidar500m":
        return [([a.numpy() for a in gen_lidar(n, 500, cpu)], 1e-4)]
    ax = [a.numpy() for a in gen_clusters(n, max(1, 32768 * n // args.particles), 0.002, 1000, cpu)]
    return [(ax, eb) for eb in (1e-2, 1e-3, 1e-4)]


def run_reference(args, world, rank):
    """--impl reference: the reference's algorithm (oracle port; the Python
    reference cannot travel to the box) on the host cores, same metric."""
    if rank != 0:
        return
    samples = reference_sample(args)
    cores = _cpu_cores()
    decomp_only = args.workload == "decomp1b"
    with make_pool(cores) as pool:
        for _ in range(args.warmup):
            cpu_oracle_round(samples, cores, pool)
        tc = td = 0.0
        nbytes = 0
        for _ in range(args.steps):
            c, d, b = cpu_oracle_round(samples, cores, pool)
            tc += c
            td += d
            nbytes += b
    v = nbytes / (td if decomp_only else tc) / 1e9
    wl = WORKLOADS[args.workload]
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": (td if decomp_only else tc) / args.steps * 1e3,
            "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (CPU-generated sample of the same generator family)",
            "config": {"workload": f"{args.workload}: {wl['desc']} (bounded CPU sample)",
                       "baseline_config": wl["config"],
                       "value_is": "decompress GB/s" if decomp_only else "compress GB/s",
                       "sample_particles_per_dataset": args.cpu_sample},
            "impl": "reference",
            "decompress": {"value": nbytes / td / 1e9, "unit": "GB/s"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "port", "cpu_model": _cpu_model(),
                             "sample": f"{args.cpu_sample} particles x {len(samples)} jobs per step, "
                                       f"oracle/gpz_oracle.py (restatement of /root/reference/pkg/src/gpz) over "
                                       f"{cores} processes"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
