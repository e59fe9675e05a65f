#!/usr/bin/env python
"""Validate and time tune candidates on corpus ops (measurement tool, GPU box):
    python tools/try_params.py --ops 42:20,41:20 --params 'BN=128,sk=0,tm=1' 'BN=128,sk=1,tm=1,cl=3'
Each candidate is checked on the device against conv_simple at the reference
tolerance (the tuner's check) and timed cold (L2 flushed, CUDA events, median
of --reps); prints us, TFLOP/s and max error per (op, candidate)."""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1611_06945_b200 import corpus, runner, tuner  # noqa: E402
from paper_1611_06945_b200.frontend import with_fused  # noqa: E402
from paper_1611_06945_b200.variants import VARIANTS, TuneParams  # noqa: E402

BASE = "MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,"

ap = argparse.ArgumentParser()
ap.add_argument("--ops", required=True, help="row:batch,...")
ap.add_argument("--params", nargs="+", required=True)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--warm", action="store_true", help="no L2 flush between reps")
a = ap.parse_args()
for spec in a.ops.split(","):
    row, batch = (int(v) for v in spec.split(":"))
    op = corpus.corpus(batch)[row]
    g = with_fused(op.graph(), "conv", "relu")
    node = g.node("conv")
    inputs = runner.node_test_inputs(node, g.edges, f"try:{row}:{batch}")
    x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
    ref = runner.ConvOp(VARIANTS["conv_simple"].generate(node, g.edges, TuneParams()), x, w, b)
    ref.launch()
    torch.cuda.synchronize()
    terms = op.in_chans * op.ksz * op.ksz
    for ptxt in a.params:
        vname = None
        if ":" in ptxt.split(",")[0]:  # "conv_wino:BN=128,..." names the variant
            vname, ptxt = ptxt.split(":", 1)
        p = TuneParams.from_string(BASE + ptxt)
        vname = vname or ("conv_fc" if (op.ksz == op.in_y and op.pad == 0 and "fc" in ptxt) else (
            "conv_1x1" if op.ksz == 1 else "conv_umma"))
        v = VARIANTS[vname]
        why = v.applies(node, g.edges, p)
        if why:
            print(f"row{row} N={batch} {ptxt}: inapplicable ({why})", flush=True)
            continue
        try:
            o = runner.ConvOp(v.generate(node, g.edges, p), x, w, b)
            o.launch()
            torch.cuda.synchronize()
            ok, err = tuner.device_compare(o.y, ref.y, tuner.tolerance_for(terms, p.prec))
            ms = o.time_ms(warmup=3, reps=a.reps, l2_flush=not a.warm)
            print(f"row{row} N={batch} {vname} {ptxt}: {ms * 1e3:8.2f} us {op.flops_computed / ms / 1e9:7.1f} TFLOP/s "
                  f"err {err:.2e} {'ok' if ok else 'FAIL'} (K={terms})", flush=True)
        except Exception as e:  # a faulting candidate: report and stop (the context is gone)
            print(f"row{row} N={batch} {ptxt}: FAILED {type(e).__name__}: {str(e)[:200]}", flush=True)
            raise
