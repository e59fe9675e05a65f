#!/usr/bin/env python
"""Launch one corpus op a few times (for ncu captures):
    python tools/run_op.py --row 42 --batch 20 [--variant conv_umma --params 'MNt=...'] [--reps 3]
Without --variant, the shipped TuneDB's choice is used."""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1611_06945_b200 import corpus, runner, tuner  # noqa: E402
from paper_1611_06945_b200.frontend import with_fused  # noqa: E402
from paper_1611_06945_b200.variants import VARIANTS, TuneParams, select_variant  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--row", type=int, required=True)
ap.add_argument("--batch", type=int, default=20)
ap.add_argument("--variant", default=None)
ap.add_argument("--params", default=None)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
op = corpus.corpus(a.batch)[a.row]
g = with_fused(op.graph(), "conv", "relu")
node = g.node("conv")
if a.variant:
    v, p = VARIANTS[a.variant], TuneParams.from_string(a.params) if a.params else VARIANTS[a.variant].default_params(node, g.edges)
else:
    v, p = select_variant(node, g.edges, tuner.load_db(tuner.shipped_db_path()))
inputs = runner.node_test_inputs(node, g.edges, "runop")
x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
o = runner.ConvOp(v.generate(node, g.edges, p), x, w, b)
for _ in range(a.reps):
    o.launch()
torch.cuda.synchronize()
ms = o.time_ms(warmup=2, reps=10, l2_flush=True)
print(f"row{a.row} N={a.batch} {v.name} {p.to_string()} {ms * 1e3:.2f} us {op.flops_computed / ms / 1e9:.1f} TFLOP/s")
