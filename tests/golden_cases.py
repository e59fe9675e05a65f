"""Loader for the reference-generated golden conv vectors (tests/golden/)."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from oracle import conv_ref

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()[:16]


def load():
    with open(os.path.join(HERE, "conv_cases.json")) as fh:
        meta = json.load(fh)
    arrays = np.load(os.path.join(HERE, "conv_cases.npz"))
    return meta["cases"], arrays


def inputs(case):
    b, ic, h, w = case["in"]
    return conv_ref.conv_inputs(b, ic, h, w, case["out_chans"], case["ksz"], case["seed"])


def expected(case, arrays):
    """(values, flat_index_step): full output or a strided sample of it."""
    if case["stored"] == "full":
        return arrays[f"{case['id']}/out"].reshape(-1), 1
    return arrays[f"{case['id']}/sample"], case["sample_step"]
