"""Loaders for the committed golden fixtures (made by tests/golden/make_golden.py
from the reference implementation)."""

import hashlib
import json
import os

import numpy as np

from cases import CASES, make_axes  # noqa: F401

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

with open(os.path.join(HERE, "golden.json")) as f:
    GOLDEN = json.load(f)
_NPZ = np.load(os.path.join(HERE, "containers.npz"))
CONTAINERS = {k: _NPZ[k].tobytes() for k in _NPZ.files}


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(a if isinstance(a, (bytes, bytearray)) else np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def case_ids():
    return [c[0] for c in CASES]


def case(name):
    for c in CASES:
        if c[0] == name:
            return c
    raise KeyError(name)


def error_prefix(msg: str) -> str:
    return msg.split(":")[0] if msg.startswith("block ") else ""

with open(os.path.join(HERE, "stress.json")) as f:
    STRESS = json.load(f)  # 1M UNIFORM_BOX / JITTERED_LATTICE goldens (tests/golden/make_golden_stress.py)
