#!/usr/bin/env python
"""Launch one op many times, synchronising (and checking vs conv_simple) after each:
    python tools/stress_op.py --row 25 --batch 20 --variant conv_umma --params '...' [--iters 50] [--flush]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1611_06945_b200 import corpus, runner  # noqa: E402
from paper_1611_06945_b200.frontend import with_fused  # noqa: E402
from paper_1611_06945_b200.variants import VARIANTS, TuneParams  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--row", type=int, required=True)
ap.add_argument("--batch", type=int, default=20)
ap.add_argument("--variant", default="conv_umma")
ap.add_argument("--params", required=True)
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--flush", action="store_true")
a = ap.parse_args()
op = corpus.corpus(a.batch)[a.row]
g = with_fused(op.graph(), "conv", "relu")
node = g.node("conv")
inputs = runner.node_test_inputs(node, g.edges, "stress")
x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
ref = runner.ConvOp(VARIANTS["conv_simple"].generate(node, g.edges, TuneParams()), x, w, b)
ref.launch()
o = runner.ConvOp(VARIANTS[a.variant].generate(node, g.edges, TuneParams.from_string(a.params)), x, w, b)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for i in range(a.iters):
    if a.flush:
        flush.zero_()
    o.y.fill_(float("nan"))
    o.launch()
    try:
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(f"row{a.row} {a.params}: FAILED at iter {i}: {e}")
        sys.exit(1)
    err = ((o.y - ref.y).abs() / ref.y.abs().clamp_min(1e-6)).max().item()
    if not err < 1e-3:
        print(f"row{a.row} {a.params}: WRONG at iter {i}: max rel err {err}")
        sys.exit(1)
print(f"row{a.row} N={a.batch} {a.params}: {a.iters} iters ok (last err {err:.2e})")
