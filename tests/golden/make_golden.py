"""Generate golden conv vectors by running the REFERENCE implementation.

Run in the build container (the reference is not shipped to the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg python tests/golden/make_golden.py

It imports the reference package ``cuclgen`` and records, per case, the op
(ksz/stride/pad/out_chans, input img:chan:y:x, fused activation), the seed
string its synthetic inputs are drawn from (runner.node_test_inputs,
cuclgen/runner.py:39-45), sha256 digests of those inputs, and the output of
the reference oracle (runner.node_reference -> oracle.ref_conv,
cuclgen/oracle.py:69-99).  Small outputs are stored whole; large ones as a
strided sample plus a digest.

Cases:
* 40 random small convs drawn with the reference test helper
  ``random_conv_case`` (pkg/tests/helpers.py:19-40), half with fused ReLU;
* all 43 corpus rows downscaled with the reference ``tuner.downscale_conv``
  (tuner.py:98-126) to <= 2e6 FLOPs;
* full-size ops: AlexNet conv1 at N=1 (config 1, corpus row 34), GoogLeNet
  5a 1x1 (row 2) at N=1, fc7 (row 13) at N=1, NiN conv4 (row 36) at N=1.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

from cuclgen import corpus as rcorpus
from cuclgen import runner as rrunner
from cuclgen import tuner as rtuner
from cuclgen.frontend import conv_graph

sys.path.insert(0, "/root/reference/pkg/tests")
from helpers import random_conv_case  # noqa: E402  (reference test helper)

HERE = os.path.dirname(os.path.abspath(__file__))
FULL_LIMIT = 6_000  # store outputs with at most this many elements whole


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()[:16]


def record(case_id, p, in_dims, seed, act, arrays, manifest):
    g = conv_graph(p, in_dims)
    if act:
        from dataclasses import replace

        g.nodes = [replace(n, fused_activation=act) if n.name == "conv" else n for n in g.nodes]
    node = g.node("conv")
    inputs = rrunner.node_test_inputs(node, g.edges, seed)
    ref = rrunner.node_reference(node, g.edges, inputs).to_np()
    x = inputs["data"].to_np()
    f = inputs["conv_filts"].to_np()
    b = inputs["conv_bias"].to_np()
    entry = {
        "id": case_id,
        "ksz": p.ksz, "stride": p.stride, "pad": p.pad, "out_chans": p.out_chans,
        "in": list(in_dims.sizes), "act": act, "seed": seed,
        "sig": rtuner.op_signature(node, g.edges),
        "x_digest": digest(x), "f_digest": digest(f), "b_digest": digest(b),
        "out_shape": list(ref.shape), "out_digest": digest(ref),
        "reduction_terms": rrunner.conv_reduction_terms(node, g.edges),
    }
    if ref.size <= FULL_LIMIT:
        arrays[f"{case_id}/out"] = ref
        entry["stored"] = "full"
    else:
        step = max(1, ref.size // 1500)
        arrays[f"{case_id}/sample"] = ref.reshape(-1)[::step]
        entry["stored"] = "sample"
        entry["sample_step"] = step
    manifest.append(entry)


def main():
    arrays, manifest = {}, []
    rng = np.random.default_rng(20240611)
    for i in range(40):
        p, dims = random_conv_case(rng, max_flops=200_000)
        record(f"rand{i:02d}", p, dims, f"golden:rand{i}", "relu" if i % 2 else None, arrays, manifest)
    for i, op in enumerate(rcorpus.corpus()):
        p2, d2 = rtuner.downscale_conv(op.conv_params, op.input_dims, 2_000_000)
        record(f"twin{i:02d}", p2, d2, f"golden:twin{i}", "relu" if i % 3 == 0 else None, arrays, manifest)
    ops = rcorpus.corpus()
    for row in (34, 2, 13, 36):
        op = ops[row]
        from cuclgen.ndarray import DimsSpec

        dims = DimsSpec.row_major(("img", "chan", "y", "x"), (1, op.in_chans, op.in_y, op.in_x))
        record(f"full{row:02d}", op.conv_params, dims, f"golden:full{row}", "relu", arrays, manifest)
    np.savez_compressed(os.path.join(HERE, "conv_cases.npz"), **arrays)
    with open(os.path.join(HERE, "conv_cases.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "cuclgen 0.1.0 (/root/reference/pkg)",
                   "cases": manifest}, fh, indent=1)
    print(f"wrote {len(manifest)} cases")


if __name__ == "__main__":
    main()
