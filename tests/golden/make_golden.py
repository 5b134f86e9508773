"""Generate the golden fixtures from the REFERENCE implementation.

Runs only in the build container, where /root/reference exists:
    python tests/golden/make_golden.py
It imports the reference package ``gpz`` from /root/reference/pkg/src, runs
it on every case of cases.py (inputs regenerated with the oracle's
generators, whose bytes are checked against the reference's own generators
here), and writes:
  golden.json      outcomes: container length + SHA-256, reconstruction
                   SHA-256, error class + "block i" prefix, bit-flip outcomes
  containers.npz   the small containers themselves (byte-level diffs)
Nothing here is imported at test time except the two output files.
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
from gpz.bench import GenKind, GenSpec, generate  # noqa: E402

from cases import CASES, make_axes  # noqa: E402
from oracle import gpz_oracle as O  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes() if not isinstance(a, (bytes, bytearray)) else a)
    return h.hexdigest()


def outcome(fn):
    try:
        return fn(), None
    except gpz.GpzError as exc:
        return None, [type(exc).__name__, str(exc)]


def check_generators():
    """The oracle's generators must reproduce the reference's bytes."""
    for kind, f in ((GenKind.GAUSSIAN_CLUSTERS, O.gen_clusters), (GenKind.UNIFORM_BOX, O.gen_uniform),
                    (GenKind.JITTERED_LATTICE, O.gen_lattice)):
        for dims in (1, 2, 3):
            for prec, op in ((gpz.Precision.F32, O.F32), (gpz.Precision.F64, O.F64)):
                ref = generate(GenSpec(kind=kind, count=5000, dims=dims, seed=dims * 7, precision=prec))
                mine = f(5000, dims=dims, seed=dims * 7, prec=op)
                assert all(np.array_equal(a, b) for a, b in zip(ref.axes, mine)), (kind, dims, prec)


def main():
    check_generators()
    out = {"cases": {}, "bitflip": {}, "big": {}}
    blobs = {}
    for (name, gen, count, dims, dt, eb, mode, bs, t, pres, seed, extra) in CASES:
        axes = make_axes(gen, count, dims, dt, seed, extra, O)
        cfg = gpz.CompressConfig(error_bound=eb, eb_mode=gpz.EbMode(mode), block_size=bs,
                                 target_segs_per_axis=t, preserve_order=pres)
        rec = {"input_sha": sha(*axes)}

        def run():
            return gpz.compress(gpz.Dataset.from_axes(axes), cfg)

        blob, err = outcome(run)
        if err is None and dt == "f32" and gen == "nonfinite":
            raise AssertionError
        rec["error"] = err
        if blob is not None:
            rec["container_len"] = len(blob)
            rec["container_sha"] = sha(blob)
            ds = gpz.decompress(blob)
            rec["recon_sha"] = sha(*ds.axes)
            blobs[name] = np.frombuffer(blob, np.uint8)
            # the oracle must agree byte for byte
            assert O.compress(axes, O.Config(eb, mode, bs, t, pres)) == blob, name
        else:
            try:
                O.compress(axes, O.Config(eb, mode, bs, t, pres))
                raise AssertionError(f"oracle accepted {name}")
            except O.OracleError as exc:
                assert type(exc).__name__ == err[0], (name, exc, err)
        out["cases"][name] = rec
        print(name, rec.get("container_len"), err)

    # every single-bit flip of a small 2D container (tests/test_container.py:198-249 style)
    rng = np.random.default_rng(88)
    axes = [rng.uniform(0, 1, 1500).astype(np.float32) for _ in range(2)]
    cfg = gpz.CompressConfig(error_bound=1e-2, block_size=512)
    blob = gpz.compress(gpz.Dataset.from_axes(axes), cfg)
    blobs["bitflip_base"] = np.frombuffer(blob, np.uint8)
    flips = []
    for pos in range(len(blob)):
        for bit in range(8):
            c = bytearray(blob)
            c[pos] ^= 1 << bit
            ds, err = outcome(lambda: gpz.decompress(bytes(c)))
            if err is None:
                flips.append([pos, bit, "ok", sha(*ds.axes)[:16]])
            else:
                blk = err[1].split(":")[0] if err[1].startswith("block ") else ""
                flips.append([pos, bit, err[0], blk])
    out["bitflip"] = {"len": len(blob), "sha": sha(blob), "outcomes": flips}
    print("bitflip outcomes", len(flips))

    # the 1M clustered fixture (tests/test_acceptance.py:180-184)
    big = O.gen_clusters(1_000_000, dims=3, seed=42)
    ref = generate(GenSpec(kind=GenKind.GAUSSIAN_CLUSTERS, count=1_000_000, dims=3, seed=42))
    assert all(np.array_equal(a, b) for a, b in zip(ref.axes, big))
    out["big"]["input_sha"] = sha(*big)
    for eb in (1e-2, 1e-3, 1e-4):
        blob = gpz.compress(ref, gpz.CompressConfig(error_bound=eb))
        rec = gpz.decompress(blob)
        out["big"][repr(eb)] = {"container_len": len(blob), "container_sha": sha(blob),
                                "recon_sha": sha(*rec.axes)}
        print("big", eb, len(blob))

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"), sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "containers.npz"), **blobs)


if __name__ == "__main__":
    main()
