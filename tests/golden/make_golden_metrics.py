"""Golden fixtures for the evaluation path (metrics.py) from the REFERENCE.

Runs only in the build container, where /root/reference exists:
    python tests/golden/make_golden_metrics.py
For every case of METRIC_CASES it builds the original dataset (the oracle's
generators, byte-identical to the reference's — checked by make_golden.py),
a reconstruction (reference compress -> decompress, then the case's
deterministic perturbation) and runs the reference's pair_blocks, nrmse,
aggregate_psnr, verify_bound and evaluate.  Writes metrics_golden.json
(pairing SHA-256, NRMSE per axis, PSNR, max error, violations, CSV row, or
the error class and message).
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import gpz  # noqa: E402  (the reference)
from gpz import metrics as M  # noqa: E402

from metric_cases import METRIC_CASES, build  # noqa: E402
from oracle import gpz_oracle as O  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    out = {}
    for case in METRIC_CASES:
        name = case["name"]
        orig, rec, cfg_kw = build(case, O, gpz)
        cfg = gpz.CompressConfig(error_bound=cfg_kw["error_bound"], eb_mode=gpz.EbMode(cfg_kw["eb_mode"]),
                                 block_size=cfg_kw["block_size"],
                                 target_segs_per_axis=cfg_kw["target_segs_per_axis"])
        dso = gpz.Dataset.from_axes(orig)
        r = {}
        try:
            dsr = gpz.Dataset.from_axes(rec)
            eb_abs = gpz.resolve_absolute_bound(dso, cfg)
            oi, ri = M.pair_blocks(dso, dsr, cfg, eb_abs)
            r["pairing_sha"] = sha(oi, ri)
            r["nrmse"] = [M.nrmse(dso.axes[a], dsr.axes[a], (oi, ri)) for a in range(dso.dims)]
            r["psnr"] = M.aggregate_psnr(r["nrmse"])
            rep = M.verify_bound(dso, dsr, eb_abs, cfg)
            r["max_err"] = rep.max_err
            r["violations"] = [list(v) for v in rep.violations]
            r["checked"] = rep.checked
            blob_len = case.get("blob_len", 1000)
            r["csv"] = M.evaluate(dso, dsr, blob_len, cfg_kw["error_bound"], eb_abs, cfg).to_csv()
            r["eb_abs"] = eb_abs
            r["error"] = None
        except gpz.GpzError as exc:
            r = {"error": [type(exc).__name__, str(exc)]}
        out[name] = r
        print(name, r.get("error") or (r["max_err"], len(r["violations"])))
    with open(os.path.join(HERE, "metrics_golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
