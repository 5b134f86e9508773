"""Synthetic particle datasets and the end-to-end throughput harness.

Mirrors the reference's ``gpz.bench`` (bench.py:1-163): the same GenKind /
GenSpec / generate / run_bench / BENCH_CSV_HEADER surface and CSV schema.

* ``generate(spec)`` reproduces the reference's datasets byte for byte (the
  same numpy Generator calls, bench.py:56-94), so a seed names the same
  particles in both packages.
* ``generate_device(spec)`` draws the same distribution families directly in
  HBM with PyTorch's Philox generator (a different random stream), for the
  280M-2B particle scales where host generation and the PCIe upload would
  dominate; every intermediate is float64 like the reference's.
* ``run_bench`` times the public compress / decompress calls end to end
  (wall clock around each call, as ``_timed``, bench.py:119-127) and scores
  the reconstruction with the GPU metrics (K5).
"""

from __future__ import annotations

import math
import statistics
import time
from dataclasses import dataclass, replace
from enum import Enum

import numpy as np

from . import metrics, pipeline
from .errors import DomainError
from .model import CompressConfig, Dataset, Precision
from .pipeline import resolve_absolute_bound

__all__ = ["GenKind", "GenSpec", "generate", "generate_device", "run_bench", "BenchRow", "bench_csv",
           "BENCH_CSV_HEADER"]


class GenKind(Enum):
    UNIFORM_BOX = "uniform"
    GAUSSIAN_CLUSTERS = "clusters"
    JITTERED_LATTICE = "lattice"


@dataclass(frozen=True)
class GenSpec:
    """One synthetic dataset (bench.py:20-50 field set).

    The box is [0, extent)^dims.  ``clusters`` / ``sigma`` shape
    GAUSSIAN_CLUSTERS (sigma in box units); ``pitch`` / ``jitter`` shape
    JITTERED_LATTICE (grid spacing, and the uniform displacement bound per
    axis).
    """

    kind: GenKind
    count: int
    dims: int = 3
    seed: int = 0
    precision: Precision = Precision.F32
    extent: float = 1.0
    clusters: int = 32
    sigma: float = 0.01
    pitch: float = 0.05
    jitter: float = 0.01

    def __post_init__(self) -> None:
        if self.count <= 0:
            raise DomainError(f"count must be positive, got {self.count}")
        if not 1 <= self.dims <= 3:
            raise DomainError(f"dims must be 1, 2 or 3, got {self.dims}")


def _lattice_side(spec: GenSpec) -> int:
    side = max(1, round(spec.count ** (1.0 / spec.dims)))
    while side**spec.dims < spec.count:
        side += 1
    return side


def generate(spec: GenSpec) -> Dataset:
    """The reference's dataset for this spec, byte for byte (bench.py:56-94)."""
    rng = np.random.default_rng(spec.seed)
    if spec.kind is GenKind.UNIFORM_BOX:
        axes = [rng.uniform(0.0, spec.extent, spec.count) for _ in range(spec.dims)]
    elif spec.kind is GenKind.GAUSSIAN_CLUSTERS:
        centers = rng.uniform(0.0, spec.extent, size=(spec.clusters, spec.dims))
        base, extra = divmod(spec.count, spec.clusters)
        sizes = np.full(spec.clusters, base, dtype=np.int64)
        sizes[:extra] += 1
        assignment = np.repeat(np.arange(spec.clusters), sizes)
        noise = rng.normal(0.0, spec.sigma, size=(spec.count, spec.dims))
        points = centers[assignment] + noise
        axes = [points[:, a] for a in range(spec.dims)]
    else:
        side = _lattice_side(spec)
        grids = np.meshgrid(*[np.arange(side, dtype=np.float64)] * spec.dims, indexing="ij")
        axes = []
        for g in grids:
            flat = g.reshape(-1)[: spec.count] * spec.pitch
            axes.append(flat + rng.uniform(-spec.jitter, spec.jitter, spec.count))
    return Dataset(axes=tuple(axes), precision=spec.precision)


def generate_device(spec: GenSpec, device=None) -> Dataset:
    """The same generator family drawn on the GPU (Philox stream; not the
    reference's bytes), for datasets too large to build on the host."""
    import torch

    dev = torch.device(device) if device is not None else pipeline._device()
    g = torch.Generator(device=dev).manual_seed(spec.seed)
    f64 = torch.float64
    n = spec.count
    if spec.kind is GenKind.UNIFORM_BOX:
        axes = [torch.rand(n, generator=g, device=dev, dtype=f64) * spec.extent for _ in range(spec.dims)]
    elif spec.kind is GenKind.GAUSSIAN_CLUSTERS:
        centers = torch.rand(spec.clusters, spec.dims, generator=g, device=dev, dtype=f64) * spec.extent
        base, extra = divmod(n, spec.clusters)
        # cluster of particle i with the reference's sizes: the first `extra` clusters hold base + 1
        i = torch.arange(n, device=dev, dtype=torch.int64)
        cut = extra * (base + 1)
        assign = torch.where(i < cut, i // (base + 1), extra + (i - cut) // max(base, 1))
        axes = [centers[assign, a] + spec.sigma * torch.randn(n, generator=g, device=dev, dtype=f64)
                for a in range(spec.dims)]
    else:
        side = _lattice_side(spec)
        i = torch.arange(n, device=dev, dtype=torch.int64)
        axes = []
        for a in range(spec.dims):
            stride = side ** (spec.dims - 1 - a)  # meshgrid "ij": the first axis varies slowest
            coord = ((i // stride) % side).to(f64) * spec.pitch
            jit = (torch.rand(n, generator=g, device=dev, dtype=f64) * 2.0 - 1.0) * spec.jitter
            axes.append(coord + jit)
    return Dataset(axes=tuple(a.to(spec.precision.torch_dtype) for a in axes), precision=spec.precision)


BENCH_CSV_HEADER = "kind,count,dims,seed,eb,cr,bitrate,psnr,comp_gbps,decomp_gbps"


@dataclass(frozen=True)
class BenchRow:
    spec: GenSpec
    eb: float
    cr: float
    bitrate: float
    psnr: float
    comp_gbps: float
    decomp_gbps: float

    def to_csv(self) -> str:
        """One line in BENCH_CSV_HEADER's column order (bench.py:108-116 formats)."""
        four = lambda v: format(v, ".4f")  # noqa: E731
        cols = [self.spec.kind.value, str(self.spec.count), str(self.spec.dims), str(self.spec.seed),
                format(self.eb, "g"), four(self.cr), four(self.bitrate),
                "inf" if math.isinf(self.psnr) else four(self.psnr),
                four(self.comp_gbps), four(self.decomp_gbps)]
        return ",".join(cols)


def _timed(fn, repetitions: int):
    """Call ``fn`` ``repetitions`` times; return (median seconds, the last
    call's value) — the reference's timing rule (bench.py:119-127)."""
    durations, out = [], None
    for _ in range(repetitions):
        t0 = time.perf_counter()
        out = fn()
        durations.append(time.perf_counter() - t0)
    return statistics.median(durations), out


def run_bench(spec: GenSpec, eb_list, cfg: CompressConfig, repetitions: int = 3, workers: int = 1,
              device_data: bool = False) -> list:
    """One BenchRow per bound (bench.py:130-163).

    ``device_data=False`` times the host API exactly like the reference
    (numpy in, bytes out, bytes in, numpy out; PCIe copies inside the
    window); ``device_data=True`` generates on the GPU and times
    compress_device / decompress_device (HBM in, HBM out).
    """
    if repetitions < 1:
        raise DomainError("repetitions must be at least 1")
    import torch

    ds = generate_device(spec) if device_data else generate(spec)
    gb = ds.nbytes / 1e9
    comp = pipeline.compress_device if device_data else pipeline.compress
    decomp = pipeline.decompress_device if device_data else pipeline.decompress

    def sync(v):
        torch.cuda.synchronize()
        return v

    rows = []
    for eb in eb_list:
        run_cfg = replace(cfg, error_bound=float(eb))
        comp_s, blob = _timed(lambda: sync(comp(ds, run_cfg)), repetitions)
        decomp_s, rec = _timed(lambda: sync(decomp(blob)), repetitions)
        eb_abs = resolve_absolute_bound(ds, run_cfg)
        nbytes = blob.numel() if device_data else len(blob)
        row = metrics.evaluate(ds, rec, nbytes, float(eb), eb_abs, run_cfg)
        rows.append(BenchRow(spec=spec, eb=float(eb), cr=row.cr, bitrate=row.bitrate, psnr=row.psnr,
                             comp_gbps=gb / comp_s if comp_s > 0 else float("inf"),
                             decomp_gbps=gb / decomp_s if decomp_s > 0 else float("inf")))
    return rows


def bench_csv(rows: list) -> str:
    return "\n".join([BENCH_CSV_HEADER, *(r.to_csv() for r in rows)]) + "\n"
