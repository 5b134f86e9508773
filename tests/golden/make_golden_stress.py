"""Generate the 1M-particle stress goldens from the REFERENCE implementation.

SURVEY.md §8(d) names two stress fixture families besides the clustered
acceptance fixture: UNIFORM_BOX (worst locality, the widest keys) and
JITTERED_LATTICE (/root/reference/pkg/src/gpz/bench.py:56-57,73-83).  This
script runs the reference package ``gpz`` (/root/reference/pkg/src, build
container only) on both at 1M particles, dims 3, float32, seed 42 and the
range-relative bounds 1e-2 / 1e-3 / 1e-4, and records container length and
SHA-256 and reconstruction SHA-256 in stress.json.  The inputs are the
reference's own generator output (GenSpec defaults), which the oracle's
generators reproduce byte for byte (checked here too).

    python tests/golden/make_golden_stress.py
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

import gpz  # noqa: E402  (the reference)
from gpz.bench import GenKind, GenSpec, generate  # noqa: E402

from oracle import gpz_oracle as O  # noqa: E402

N = 1_000_000
SEED = 42
EBS = (1e-2, 1e-3, 1e-4)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(a if isinstance(a, (bytes, bytearray)) else np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    out = {}
    for kind, gen in ((GenKind.UNIFORM_BOX, O.gen_uniform), (GenKind.JITTERED_LATTICE, O.gen_lattice)):
        ref = generate(GenSpec(kind=kind, count=N, dims=3, seed=SEED))
        mine = gen(N, dims=3, seed=SEED)
        assert all(np.array_equal(a, b) for a, b in zip(ref.axes, mine)), kind
        rec = {"input_sha": sha(*ref.axes)}
        for eb in EBS:
            blob = gpz.compress(ref, gpz.CompressConfig(error_bound=eb))
            dec = gpz.decompress(blob)
            rec[repr(eb)] = {"container_len": len(blob), "container_sha": sha(blob), "recon_sha": sha(*dec.axes)}
            print(kind.value, eb, len(blob), flush=True)
        out[kind.value] = rec
    with open(os.path.join(HERE, "stress.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
