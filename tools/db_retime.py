#!/usr/bin/env python
"""Re-time the shipped TuneDB's choices on the current library (GPU box):
for every sweep op, the DB's (variant, params) is checked on the device against
conv_simple at the mode's tolerance and timed cold (L2 flushed, CUDA events),
and printed beside the cost the DB recorded when it was tuned.

    python tools/db_retime.py [--prec 0] [--batches 1,5,20] [--only-bn 32,64] [--csv out.csv]
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1611_06945_b200 import corpus, runner, tuner  # noqa: E402
from paper_1611_06945_b200.frontend import with_fused  # noqa: E402
from paper_1611_06945_b200.variants import VARIANTS, TuneParams, select_variant  # noqa: E402

DBS = {0: "tunedb_b200_fp32.tsv", 1: "tunedb_b200_bf16.tsv", 2: "tunedb_b200_fp8.tsv"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prec", type=int, default=0)
    ap.add_argument("--batches", default="1,5,20")
    ap.add_argument("--only-bn", default=None, help="only ops whose chosen BN is in this list")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--csv", default=None)
    a = ap.parse_args()
    db = tuner.load_db(os.path.join(os.path.dirname(tuner.shipped_db_path()), DBS[a.prec]))
    only = {int(v) for v in a.only_bn.split(",")} if a.only_bn else None
    rows, old_sum, new_sum = [], 0.0, 0.0
    for row, op in corpus.sweep_ops(tuple(int(b) for b in a.batches.split(","))):
        g = with_fused(op.graph(), "conv", "relu")
        node = g.node("conv")
        v, p = select_variant(node, g.edges, db, prec=a.prec)
        if only is not None and p.bn not in only:
            continue
        rec = db.records.get(tuner.op_signature(node, g.edges))
        inputs = runner.node_test_inputs(node, g.edges, f"retime:{row}:{op.batch}")
        x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
        ref = runner.ConvOp(VARIANTS["conv_simple"].generate(node, g.edges, TuneParams()), x, w, b)
        o = runner.ConvOp(v.generate(node, g.edges, p), x, w, b)
        ref.launch()
        o.launch()
        torch.cuda.synchronize()
        ok, err = tuner.device_compare(o.y, ref.y, tuner.tolerance_for(op.in_chans * op.ksz * op.ksz, p.prec))
        us = o.time_ms(warmup=3, reps=a.reps, l2_flush=True) * 1e3
        old = rec.cost * 1e-3 if rec is not None else float("nan")
        old_sum += old if rec is not None else 0.0
        new_sum += us
        line = f"{row},{op.batch},{v.name},\"{p.to_string()}\",{old:.2f},{us:.2f},{err:.2e},{'ok' if ok else 'FAIL'}"
        rows.append(line)
        print(f"row{row:2d} N={op.batch:2d} {v.name:15s} BN={p.bn:3d} db {old:8.2f} us  now {us:8.2f} us  "
              f"x{old / us if us else 0:5.2f}  err {err:.2e} {'ok' if ok else 'FAIL'}", flush=True)
        del ref, o, x, w, b
    print(f"total: db {old_sum:.1f} us  now {new_sum:.1f} us  ({len(rows)} ops)")
    if a.csv:
        with open(a.csv, "w") as fh:
            fh.write("row,n,variant,params,db_us,now_us,max_err,check\n" + "\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
