"""The package's bench module (gpz.bench mirror): generators and run_bench.

CPU: ``generate`` reproduces the reference's generators byte for byte (the
oracle's generators are checked against the reference itself by
tests/golden/make_golden.py).  GPU: ``generate_device`` draws the same
families in HBM, and ``run_bench`` produces rows in the reference's CSV
schema.
"""

import math

import numpy as np
import pytest

from oracle import gpz_oracle as O

gz = pytest.importorskip("paper_2508_10305_b200")
from paper_2508_10305_b200 import bench as B  # noqa: E402


@pytest.mark.parametrize("kind,fn", [(B.GenKind.GAUSSIAN_CLUSTERS, O.gen_clusters),
                                     (B.GenKind.UNIFORM_BOX, O.gen_uniform),
                                     (B.GenKind.JITTERED_LATTICE, O.gen_lattice)])
@pytest.mark.parametrize("dims", [1, 2, 3])
@pytest.mark.parametrize("prec", [gz.Precision.F32, gz.Precision.F64])
def test_generate_matches_reference_bytes(kind, fn, dims, prec):
    ds = B.generate(B.GenSpec(kind=kind, count=3001, dims=dims, seed=dims + 40, precision=prec))
    want = fn(3001, dims=dims, seed=dims + 40, prec=O.F32 if prec is gz.Precision.F32 else O.F64)
    assert ds.precision is prec and ds.dims == dims
    for a, b in zip(ds.axes, want):
        assert a.dtype == b.dtype and np.array_equal(a, b)


def test_genspec_validation_and_csv_row():
    with pytest.raises(gz.DomainError, match="count must be positive"):
        B.GenSpec(kind=B.GenKind.UNIFORM_BOX, count=0)
    with pytest.raises(gz.DomainError, match="dims must be 1, 2 or 3"):
        B.GenSpec(kind=B.GenKind.UNIFORM_BOX, count=5, dims=4)
    row = B.BenchRow(spec=B.GenSpec(kind=B.GenKind.GAUSSIAN_CLUSTERS, count=10, seed=3), eb=1e-3, cr=7.5,
                     bitrate=4.25, psnr=math.inf, comp_gbps=1.5, decomp_gbps=2.0)
    assert row.to_csv() == "clusters,10,3,3,0.001,7.5000,4.2500,inf,1.5000,2.0000"
    assert B.bench_csv([row]).splitlines()[0] == B.BENCH_CSV_HEADER


gpu = pytest.mark.gpu


def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@gpu
def test_generate_device_families():
    torch = _cuda()
    n = 100_003
    cl = B.generate_device(B.GenSpec(kind=B.GenKind.GAUSSIAN_CLUSTERS, count=n, dims=3, seed=9, clusters=7,
                                     sigma=1e-3))
    assert cl.on_device and cl.count == n and cl.axes[0].dtype == torch.float32
    # cluster-contiguous: the reference's sizes (first count % clusters clusters one larger)
    x = cl.axes[0].double().cpu().numpy()
    base, extra = divmod(n, 7)
    sizes = [base + 1] * extra + [base] * (7 - extra)
    starts = np.cumsum([0] + sizes)
    for c in range(7):
        seg = x[starts[c]:starts[c + 1]]
        assert seg.std() < 5e-3
    lat = B.generate_device(B.GenSpec(kind=B.GenKind.JITTERED_LATTICE, count=1000, dims=3, seed=2,
                                      precision=gz.Precision.F64))
    ref = O.gen_lattice(1000, dims=3, seed=2, prec=O.F64, jitter=0.0)
    for a, b in zip(lat.axes, ref):
        assert np.abs(a.cpu().numpy() - b).max() <= 0.01 + 1e-12
    un = B.generate_device(B.GenSpec(kind=B.GenKind.UNIFORM_BOX, count=n, dims=2, seed=1, extent=2.0))
    assert float(un.axes[1].min()) >= 0.0 and float(un.axes[1].max()) <= 2.0


@gpu
@pytest.mark.parametrize("device_data", [False, True])
def test_run_bench_rows(device_data):
    _cuda()
    spec = B.GenSpec(kind=B.GenKind.GAUSSIAN_CLUSTERS, count=200_000, dims=3, seed=42)
    rows = B.run_bench(spec, [1e-2, 1e-3], gz.CompressConfig(error_bound=1e-3), repetitions=2,
                       device_data=device_data)
    assert [r.eb for r in rows] == [1e-2, 1e-3]
    for r in rows:
        assert r.cr > 1.0 and r.comp_gbps > 0 and r.decomp_gbps > 0 and math.isfinite(r.psnr)
        assert r.to_csv().startswith("clusters,200000,3,42,")
    if not device_data:
        # the host path measures the reference's own dataset: CR equals the oracle's container ratio
        ds = B.generate(spec)
        blob = O.compress(list(ds.axes), O.Config(1e-3))
        assert rows[1].cr == pytest.approx(ds.nbytes / len(blob), rel=0, abs=1e-12)
