#!/usr/bin/env python
"""Run one (case, variant, params) on the device in isolation and report (debug):
    python tools/probe_one.py --case twin00 --variant conv_umma --params 'MNt=...'"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import conv_ref  # noqa: E402
from paper_1611_06945_b200 import runner  # noqa: E402
from paper_1611_06945_b200.frontend import ConvParams, conv_graph  # noqa: E402
from paper_1611_06945_b200.ndarray import DimsSpec  # noqa: E402
from paper_1611_06945_b200.variants import VARIANTS, TuneParams  # noqa: E402
from tests import golden_cases  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", required=True)
ap.add_argument("--variant", default="conv_umma")
ap.add_argument("--params", required=True)
a = ap.parse_args()
cases, _ = golden_cases.load()
c = [c for c in cases if c["id"] == a.case][0]
g = conv_graph(ConvParams(c["ksz"], c["stride"], c["pad"], c["out_chans"]), DimsSpec.row_major(("img", "chan", "y", "x"), c["in"]))
x, f, b = golden_cases.inputs(c)
p = TuneParams.from_string(a.params)
op = runner.ConvOp(VARIANTS[a.variant].generate(g.node("conv"), g.edges, p), *(torch.from_numpy(t).cuda() for t in (x, f, b)))
op.launch()
torch.cuda.synchronize()
want = conv_ref.ref_conv(x, f, b, c["stride"], c["pad"])
r = conv_ref.compare(op.y.cpu().numpy(), want, conv_ref.tolerance_for(c["reduction_terms"]))
print(a.case, a.params, "ok" if r.ok else "MISMATCH", r.max_rel_err)
