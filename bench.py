#!/usr/bin/env python
"""GPZ B200 compress / decompress throughput (BASELINE.json configs[1]).

Workload ("HACC-like"): per GPU, 280M particles x 6 float32
fields stored as two dims=3 datasets (positions xyz, velocities vxvyvz), each
compressed with its own range-relative bound 1e-3, block_size 1024, target 32.
Synthetic data (no network): 8192 Gaussian clusters stored cluster by
cluster; positions sigma 0.002 in the unit box, velocities = per-cluster bulk
N(0, 0.3) + per-particle N(0, 0.05); generated on the GPU from fixed seeds.

A step = compress both datasets, then decompress both containers.  `value`
is compress GB/s (input bytes / device time of the full compress_device
call, inputs resident in HBM, max over ranks); the decompress numbers ride in
the `decompress` object.  Inputs (6.72 GB) exceed L2, so no flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gpzb|reference]
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


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["gpzb", "reference"], default="gpzb")
    p.add_argument("--particles", type=int, default=PARTICLES, help="particles per GPU per dataset")
    p.add_argument("--cpu-sample", type=int, default=CPU_SAMPLE)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--compress-only", action="store_true", help="experiments: skip decompress")
    p.add_argument("--per-call", action="store_true",
                   help="one compress_device / decompress_device call per field instead of the batched calls")
    return p.parse_args()


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


def _enc_chunk(args):
    from oracle import gpz_oracle as O

    axes, eb_abs, bs = args
    return [O.encode_block([a[s:s + bs] for a in axes], eb_abs, O.Config(1e-3, block_size=bs), O.F32)
            for s in range(0, axes[0].size, bs)]


def _dec_chunk(args):
    from oracle import gpz_oracle as O

    payloads, h = args
    return [O.decode_block(p, h) for p in payloads]


def cpu_oracle_round(samples, cores, pool):
    """Oracle (the reference's algorithm restated, oracle/gpz_oracle.py) on the
    host: compress + decompress of each sample dataset, blocks spread over
    `cores` processes.  Returns (compress_s, decompress_s, bytes)."""
    from oracle import gpz_oracle as O

    bs = 1024
    t_c = t_d = 0.0
    nbytes = 0
    for axes in samples:
        n = axes[0].size
        nb = (n + bs - 1) // bs
        per = (nb + cores - 1) // cores
        t0 = time.perf_counter()
        eb_abs = O.absolute_bound(axes, O.Config(1e-3))
        jobs = [([a[i * per * bs:(i + 1) * per * bs] for a in axes], eb_abs, bs) for i in range(cores)
                if i * per * bs < n]
        payloads = [p for part in pool.map(_enc_chunk, jobs) for p in part]
        blob = O.assemble(3, O.F32, O.Config(1e-3), eb_abs, n, payloads)
        t1 = time.perf_counter()
        h, table, pay = O.read_container(blob)
        jobs = [([pay[int(table[j]):int(table[j + 1])] for j in range(i * per, min((i + 1) * per, nb))], h)
                for i in range(cores) if i * per < nb]
        parts = pool.map(_dec_chunk, jobs)
        _ = [np.concatenate([b[a] for part in parts for b in part]) for a in range(3)]
        t2 = time.perf_counter()
        t_c += t1 - t0
        t_d += t2 - t1
        nbytes += n * 3 * 4
    return t_c, t_d, nbytes


def make_pool(cores):
    import multiprocessing as mp

    return mp.get_context("fork").Pool(cores)


# ------------------------------------------------------------------ main
def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.particles
    if world > 1 and rank < world - 1:
        # shards must be block-aligned (sharded.py): every rank but the last
        # rounds its particle count up to whole 1024-particle blocks
        n = (n + 1023) // 1024 * 1024

    if args.impl == "reference":
        return run_reference(args, world, rank)

    # GPZB_BENCH_SHARE_GPU=1: every rank on cuda:0 over gloo (exercises the
    # sharded path on a one-GPU box; never used for reported numbers)
    share = os.environ.get("GPZB_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    import paper_2508_10305_b200 as gz
    from paper_2508_10305_b200 import sharded

    pos, vel = gen_hacc(n, 280 + 1000 * rank, dev)
    datasets = [gz.Dataset.from_axes(pos), gz.Dataset.from_axes(vel)]
    in_bytes = sum(d.nbytes for d in datasets)
    cfg = gz.CompressConfig(error_bound=1e-3)

    def one_step_batch(timing=None):
        """Both fields of the snapshot per call, one CUDA stream each (the
        range pass of one overlaps the encoder of the other)."""
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        c = torch.cuda.Event(enable_timing=True)
        a.record()
        if world > 1:  # this rank's shard of each field; scalar exchanges batched over the fields
            conts = sharded.compress_batch_device(datasets, cfg, timing=timing)
        else:
            conts = gz.compress_batch_device(datasets, cfg, timing=timing)
        b.record()
        if args.compress_only:
            recs = None
        elif world > 1:
            recs = sharded.decompress_batch_device(conts, timing=timing)
        else:
            recs = gz.decompress_batch_device(conts, timing=timing)
        c.record()
        torch.cuda.synchronize()
        sizes = [x.local_bytes if world > 1 else x.numel() for x in conts]
        del conts, recs
        return a.elapsed_time(b) / 1e3, b.elapsed_time(c) / 1e3, sizes

    def one_step(timing=None):
        if not args.per_call:
            return one_step_batch(timing)
        sizes, recs = [], []
        tc = td = 0.0
        for ds in datasets:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            c = torch.cuda.Event(enable_timing=True)
            a.record()
            if world > 1:
                cont = sharded.compress_device(ds, cfg, timing=timing)
            else:
                cont = gz.compress_device(ds, cfg, timing=timing)
            b.record()
            if args.compress_only:
                rec = None
            elif world > 1:
                rec = sharded.decompress_device(cont, timing=timing)
            else:
                rec = gz.decompress_device(cont, timing=timing)
            c.record()
            torch.cuda.synchronize()
            tc += a.elapsed_time(b) / 1e3
            td += b.elapsed_time(c) / 1e3
            sizes.append(cont.local_bytes if hasattr(cont, "local_bytes") else cont.numel())
            recs.append(rec)
            del cont, rec
        return tc, td, sizes

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
    t_c, t_d = sum(tcs), sum(tds)
    if world > 1:
        import torch.distributed as dist

        cdev = "cpu" if share else dev
        t = torch.tensor([t_c, t_d], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_c, t_d = t.tolist()
        z = torch.tensor([float(sum(sizes)), float(in_bytes)], dtype=torch.float64, device=cdev)
        dist.all_reduce(z)
        total_container, job_bytes = z.tolist()
    else:
        total_container = float(sum(sizes))
        job_bytes = float(in_bytes)
    steps = args.steps
    comp_gbps = job_bytes * steps / t_c / 1e9
    decomp_gbps = job_bytes * steps / t_d / 1e9
    cr = job_bytes / total_container

    # dominant-kernel rooflines from the live CUDA events
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_kind = "measured" if "hbm_gbs" in peaks else "fallback"

    def kern_ms(key):
        ev = timing.get(key, [])
        return [a.elapsed_time(b) for a, b in ev]

    enc_ms = kern_ms("encode")
    dec_ms = kern_ms("decode")
    rng_ms = kern_ms("range")
    local_in = in_bytes / len(datasets)
    local_cont = [s for s in sizes]
    enc_bytes = sum(local_in + c for c in local_cont) / len(local_cont)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(tfile):
        with open(tfile) as f:
            tj = json.load(f)
        traffic = tj.get("encode", {}).get("dram_bytes_per_launch")
    enc_avg = statistics.mean(enc_ms) / 1e3 if enc_ms else float("nan")
    dec_avg = statistics.mean(dec_ms) / 1e3 if dec_ms else float("nan")
    t_d = t_d or float("nan")
    rng_avg = statistics.mean(rng_ms) / 1e3 if rng_ms else float("nan")
    roof = {"bound": "hbm", "kernel": "encode call: k_encode / k_encode_warp (K2) + k_scan_sizes + k_copy_payloads (K3); "
                                      "batched step: durations include the other field's overlapping kernels", "achieved": enc_bytes / enc_avg / 1e9, "peak": hbm,
            "unit": "GB/s", "frac": enc_bytes / enc_avg / 1e9 / hbm, "traffic": traffic,
            "algorithmic_bytes_per_launch": enc_bytes, "avg_launch_ms": enc_avg * 1e3,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"}
    step_roof = {"compress_frac": (2 * in_bytes + total_container / world) * steps / (t_c) / 1e9 / hbm,
                 "decompress_frac": (in_bytes + total_container / world) * steps / (t_d) / 1e9 / hbm}

    line = {
        "metric": METRIC,
        "value": comp_gbps,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": t_c / steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (GPU-generated Gaussian-cluster HACC-like snapshot, fixed seeds)",
        "config": {"workload": "HACC-like 280M particles x 6 float32 fields (x,y,z,vx,vy,vz) per GPU, "
                               "two dims=3 datasets, rel-eb 1e-3, block 1024, target 32",
                   "particles_per_gpu": n, "datasets": ["pos", "vel"], "input_bytes_per_gpu": in_bytes,
                   "l2": "inputs 6.72 GB >> 126 MB L2, no flush needed",
                   "input_checksum_rank0": checksum(pos + vel)},
        "compression_ratio": cr,
        "decompress": {"value": decomp_gbps, "unit": "GB/s", "ms_per_step": t_d / steps * 1e3,
                       "roofline": {"bound": "hbm", "kernel": "decode call: k_decode_plan (K4a) + k_decode (K4)",
                                    "achieved": (local_in + statistics.mean(local_cont)) / dec_avg / 1e9,
                                    "peak": hbm, "unit": "GB/s",
                                    "frac": (local_in + statistics.mean(local_cont)) / dec_avg / 1e9 / hbm,
                                    "avg_launch_ms": dec_avg * 1e3}},
        "roofline": roof,
        "step_roofline": step_roof,
        "kernels": {"k_range_ms": rng_avg * 1e3,
                    "per_dataset_ms": {k: [statistics.mean(v[i::len(datasets)]) if v else None
                                           for i in range(len(datasets))]
                                       for k, v in (("k_encode", enc_ms), ("k_decode", dec_ms), ("k_range", rng_ms))},
                    "k_range_gbps": local_in / rng_avg / 1e9 if rng_ms else None,
                    "k_encode_ms": enc_avg * 1e3, "k_decode_ms": dec_avg * 1e3},
        "gpu_launches": launches,
        "clocks": clk.summary,
    }
    if world == 1 and not args.per_call:
        # the batched step overlaps the two fields' kernels; per-call timings
        # (untimed, after the timed region) give each kernel's own duration
        iso: dict = {}
        for _ in range(2):
            for ds in datasets:
                c1 = gz.compress_device(ds, cfg, timing=iso)
                if not args.compress_only:
                    gz.decompress_device(c1, timing=iso)
                del c1
        torch.cuda.synchronize()
        iso_ms = {k: [statistics.mean([a.elapsed_time(b) for a, b in v][i::len(datasets)])
                      for i in range(len(datasets))] for k, v in iso.items()}
        enc_iso = statistics.mean(iso_ms["encode"]) / 1e3
        line["roofline_isolated"] = {
            "note": "per-call kernel durations (one field at a time), outside the timed region",
            "per_dataset_ms": iso_ms,
            "encode_call_frac": enc_bytes / enc_iso / 1e9 / hbm,
            "decode_call_frac": ((local_in + statistics.mean(local_cont)) / (statistics.mean(iso_ms["decode"]) / 1e3)
                                 / 1e9 / hbm) if "decode" in iso_ms else None,
            "k_range_frac": local_in / (statistics.mean(iso_ms["range"]) / 1e3) / 1e9 / hbm,
        }
    if rank == 0 and not args.no_e2e:
        line["e2e"] = e2e_numbers(gz, datasets, cfg, args, in_bytes)
        line["decompress"]["e2e"] = line["e2e"].pop("decompress")
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(datasets, args.cpu_sample)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def e2e_numbers(gz, datasets, cfg, args, in_bytes):
    """The same metric through the public API from pinned HOST buffers:
    H2D of the inputs, compress, D2H of the container to Python bytes; then
    decompress(bytes) -> numpy (H2D container, decode, D2H of the axes)."""
    host = [gz.Dataset.from_axes([a.cpu().pin_memory() for a in ds.axes]) for ds in datasets]
    torch.cuda.synchronize()
    blobs = [gz.compress(h, cfg) for h in host]  # warm-up
    for b in blobs:
        gz.decompress(b)
    tc = td = 0.0
    reps = max(1, min(args.steps, 3))
    cbytes = 0
    for _ in range(reps):
        for h in host:
            t0 = time.perf_counter()
            blob = gz.compress(h, cfg)
            t1 = time.perf_counter()
            gz.decompress(blob)
            t2 = time.perf_counter()
            tc += t1 - t0
            td += t2 - t1
            cbytes += len(blob)
    return {"value": in_bytes * reps / tc / 1e9, "unit": "GB/s", "h2d_bytes_per_step": in_bytes,
            "d2h_bytes_per_step": cbytes // reps, "reps": reps,
            "api": "paper_2508_10305_b200.compress(Dataset of pinned CPU tensors) -> bytes",
            "decompress": {"value": in_bytes * reps / td / 1e9, "unit": "GB/s",
                           "h2d_bytes_per_step": cbytes // reps, "d2h_bytes_per_step": in_bytes,
                           "api": "paper_2508_10305_b200.decompress(bytes) -> numpy Dataset"}}


def cpu_baseline(datasets, sample):
    samples = [[a[:sample].cpu().numpy() for a in ds.axes] for ds in datasets]
    cores = _cpu_cores()
    with make_pool(cores) as pool:
        t_c, t_d, nbytes = cpu_oracle_round(samples, cores, pool)
    return {"value": nbytes / t_c / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
            "decompress_value": nbytes / t_d / 1e9,
            "sample": f"first {sample} particles of each of the 2 datasets ({nbytes} bytes), oracle/gpz_oracle.py "
                      f"per-block encode/decode spread over {cores} processes"}


def run_reference(args, world, rank):
    """--impl reference: the reference's algorithm (oracle port; the Python
    reference cannot travel to the box) on the host cores, same metric."""
    if rank != 0:
        return
    sample = args.cpu_sample
    g = torch.Generator().manual_seed(280)
    # same generator family as gen_hacc, on the CPU, bounded sample per dataset
    import math

    n = sample
    k = max(1, int(math.ceil(CLUSTERS * sample / PARTICLES)))
    centers = torch.rand(k, 3, generator=g, dtype=torch.float64)
    bulk = 0.3 * torch.randn(k, 3, generator=g, dtype=torch.float64)
    assign = (torch.arange(n, dtype=torch.int64) * k) // n
    pos = [(centers[assign, a] + 0.002 * torch.randn(n, generator=g, dtype=torch.float64)).float().numpy()
           for a in range(3)]
    vel = [(bulk[assign, a] + 0.05 * torch.randn(n, generator=g, dtype=torch.float64)).float().numpy()
           for a in range(3)]
    cores = _cpu_cores()
    with make_pool(cores) as pool:
        for _ in range(args.warmup):
            cpu_oracle_round([pos, vel], cores, pool)
        tc = td = 0.0
        nbytes = 0
        for _ in range(args.steps):
            c, d, b = cpu_oracle_round([pos, vel], cores, pool)
            tc += c
            td += d
            nbytes += b
    v = nbytes / tc / 1e9
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tc / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (CPU-generated sample of the same Gaussian-cluster family)",
            "config": {"workload": "HACC-like 280M particles x 6 float32 fields, rel-eb 1e-3 (bounded CPU sample)",
                       "sample_particles_per_dataset": sample},
            "impl": "reference",
            "decompress": {"value": nbytes / td / 1e9, "unit": "GB/s"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "port",
                             "sample": f"{sample} particles x 2 datasets per step, oracle/gpz_oracle.py "
                                       f"(restatement of /root/reference/pkg/src/gpz) over {cores} processes"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
