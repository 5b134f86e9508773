"""Evaluation path (metrics.py): block pairing, NRMSE, PSNR, bound check.

CPU tests pin the oracle's restatement (oracle/gpz_oracle.py) to the
reference's own outcomes (tests/golden/metrics_golden.json, made by
tests/golden/make_golden_metrics.py).  GPU tests run the K5 kernels through
the package's public metrics API against the same goldens and the oracle.
"""

import hashlib
import json
import math
import os

import numpy as np
import pytest

from metric_cases import METRIC_CASES, build
from oracle import gpz_oracle as O

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
with open(os.path.join(HERE, "metrics_golden.json")) as f:
    MGOLD = json.load(f)

NAMES = [c["name"] for c in METRIC_CASES]
CASE = {c["name"]: c for c in METRIC_CASES}
RTOL = 1e-12  # float64 sums in a different order than numpy's pairwise summation


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _oracle_outcome(case):
    orig, rec, kw = build(case, O)
    try:
        O.check_axes(orig)
        if len(rec) != len(orig) or rec[0].size != orig[0].size:
            raise O.DomainError("datasets differ in shape, cannot pair")
        O.check_axes(rec)
        eb_abs = O.absolute_bound(orig, O.Config(kw["error_bound"], eb_mode=kw["eb_mode"]))
        oi, ri = O.pair_blocks(orig, rec, kw["block_size"], kw["target_segs_per_axis"], eb_abs)
        nr = [O.nrmse(orig[a], rec[a], (oi, ri)) for a in range(len(orig))]
        m, v, ch = O.verify_bound(orig, rec, eb_abs, kw["block_size"], kw["target_segs_per_axis"])
        return dict(pairing_sha=_sha(oi, ri), nrmse=nr, psnr=O.aggregate_psnr(nr), max_err=m,
                    violations=[list(x) for x in v], checked=ch, error=None)
    except O.OracleError as exc:
        return dict(error=[type(exc).__name__, str(exc)])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_metrics(name):
    want, got = MGOLD[name], _oracle_outcome(CASE[name])
    if want["error"]:
        assert got["error"] is not None and got["error"][0] == want["error"][0]
        if want["error"][0] == "DomainError":
            assert got["error"][1] == want["error"][1]
        return
    assert got["error"] is None, got["error"]
    assert got["pairing_sha"] == want["pairing_sha"]
    assert got["max_err"] == want["max_err"]
    assert got["violations"] == want["violations"]
    assert got["checked"] == want["checked"]
    np.testing.assert_allclose(got["nrmse"], want["nrmse"], rtol=RTOL, atol=0)


# ------------------------------------------------------------------ GPU (K5)
gpu = pytest.mark.gpu


def _gz():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2508_10305_b200 as gz

    return gz


def _cfg(gz, kw):
    return gz.CompressConfig(error_bound=kw["error_bound"], eb_mode=gz.EbMode(kw["eb_mode"]),
                             block_size=kw["block_size"], target_segs_per_axis=kw["target_segs_per_axis"])


@gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_metrics_match_reference(name):
    gz = _gz()
    from paper_2508_10305_b200 import metrics as M

    case, want = CASE[name], MGOLD[name]
    orig, rec, kw = build(case, O)
    cfg = _cfg(gz, kw)
    dso = gz.Dataset.from_axes(orig)
    try:
        dsr = gz.Dataset.from_axes(rec)
        eb_abs = gz.resolve_absolute_bound(dso, cfg)
        oi, ri = M.pair_blocks(dso, dsr, cfg, eb_abs)
        nr = [M.nrmse(dso.axes[a], dsr.axes[a], (oi, ri)) for a in range(dso.dims)]
        rep = M.verify_bound(dso, dsr, eb_abs, cfg)
        row = M.evaluate(dso, dsr, case.get("blob_len", 1000), kw["error_bound"], eb_abs, cfg)
        err = None
    except gz.GpzError as exc:
        err = [type(exc).__name__, str(exc)]
    if want["error"]:
        assert err is not None and err[0] == want["error"][0], err
        if want["error"][0] == "DomainError":
            assert err[1] == want["error"][1]
        return
    assert err is None, err
    assert eb_abs == want["eb_abs"]
    assert _sha(oi, ri) == want["pairing_sha"]
    np.testing.assert_allclose(nr, want["nrmse"], rtol=RTOL, atol=0)
    assert rep.max_err == want["max_err"]
    assert [list(v) for v in rep.violations] == want["violations"]
    assert rep.checked == want["checked"]
    assert rep.ok == (not want["violations"])
    # the CSV row: identical up to the last printed digit of the float64 sums
    got_f, want_f = row.to_csv().split(","), want["csv"].split(",")
    assert got_f[:4] == want_f[:4] and got_f[-1] == want_f[-1]
    assert math.isclose(row.psnr, want["psnr"], rel_tol=1e-9) or (math.isinf(row.psnr) and math.isinf(want["psnr"]))


@gpu
def test_gpu_pairing_matches_oracle_at_scale():
    """1M clustered particles, eb 1e-3 and 1e-4: the full pairing and the bound report."""
    gz = _gz()
    from paper_2508_10305_b200 import metrics as M

    axes = O.gen_clusters(1_000_000, dims=3, seed=42)
    for eb in (1e-3, 1e-4):
        cfg = gz.CompressConfig(error_bound=eb)
        ds = gz.Dataset.from_axes(axes)
        rec = gz.decompress(gz.compress(ds, cfg))
        eb_abs = gz.resolve_absolute_bound(ds, cfg)
        oi, ri = M.pair_blocks(ds, rec, cfg, eb_abs)
        woi, wri = O.pair_blocks(axes, list(rec.axes), 1024, 32, eb_abs)
        assert np.array_equal(oi, woi) and np.array_equal(ri, wri)
        rep = M.verify_bound(ds, rec, eb_abs, cfg)
        assert rep.ok and rep.max_err <= eb_abs
        m, v, _ = O.verify_bound(axes, list(rec.axes), eb_abs, 1024, 32)
        assert rep.max_err == m and v == []


@gpu
@pytest.mark.parametrize("bs", [2048, 8192])
def test_gpu_pairing_block_size_above_1024(bs):
    """K5a's slice-based variant for blocks above 1024 particles: the
    pairing and the bound report equal the oracle's (metrics.py:49-152)."""
    gz = _gz()
    from paper_2508_10305_b200 import metrics as M

    axes = O.gen_clusters(5 * bs + 333, dims=3, seed=bs)
    cfg = gz.CompressConfig(error_bound=1e-3, block_size=bs)
    ds = gz.Dataset.from_axes(axes)
    rec = gz.decompress(gz.compress(ds, cfg))
    eb_abs = gz.resolve_absolute_bound(ds, cfg)
    oi, ri = M.pair_blocks(ds, rec, cfg, eb_abs)
    woi, wri = O.pair_blocks(axes, list(rec.axes), bs, 32, eb_abs)
    assert np.array_equal(oi, woi) and np.array_equal(ri, wri)
    rep = M.verify_bound(ds, rec, eb_abs, cfg)
    m, v, _ = O.verify_bound(axes, list(rec.axes), eb_abs, bs, 32)
    assert rep.ok and rep.max_err == m and v == []


@gpu
def test_gpu_nrmse_unpaired_and_device_inputs():
    gz = _gz()
    import torch
    from paper_2508_10305_b200 import metrics as M

    rng = np.random.default_rng(5)
    a = rng.normal(size=100_003)
    b = a + rng.normal(scale=1e-3, size=a.size)
    want = O.nrmse(a, b)
    assert math.isclose(M.nrmse(a, b), want, rel_tol=RTOL)
    assert math.isclose(M.nrmse(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()), want, rel_tol=RTOL)
    assert M.nrmse(np.zeros(0), np.zeros(0)) == 0.0
    with pytest.raises(gz.DomainError, match="degenerate field range"):
        M.nrmse(np.ones(10), np.ones(10) * 2)
    assert M.aggregate_psnr([0.0, 0.0]) == math.inf


@gpu
def test_gpu_nrmse_rejects_mismatched_inputs_like_numpy():
    """Unequal lengths and out-of-range / short pairings raise like the
    reference's numpy indexing (metrics.py:90-97) instead of reading past a
    buffer; negative indices count from the end."""
    _gz()
    from paper_2508_10305_b200 import metrics as M

    rng = np.random.default_rng(6)
    a = rng.normal(size=1000)
    b = a + rng.normal(scale=1e-3, size=a.size)
    with pytest.raises(ValueError):
        M.nrmse(a, b[:999])
    with pytest.raises(ValueError):
        M.nrmse(a, b, (np.arange(10), np.arange(9)))
    with pytest.raises(IndexError):
        M.nrmse(a, b, (np.arange(10), np.arange(10) + 995))
    p = (np.array([-1, 3, 5]), np.array([999, -997, 5]))
    assert math.isclose(M.nrmse(a, b, p), O.nrmse(a, b, p), rel_tol=RTOL)
    p = (np.arange(500), np.arange(500))
    assert math.isclose(M.nrmse(a, b, p), O.nrmse(a, b, p), rel_tol=RTOL)
