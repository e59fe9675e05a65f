#!/usr/bin/env python
"""Autotune every op of the conv sweep on the local B200 and write a TuneDB.

This is the B200 form of ``cuclgen tune`` (cli.py:125-140): one on-device
sweep per distinct op signature (tuner.tune_all), objective ``wall``.  The
result is shipped as paper_1611_06945_b200/data/tunedb_b200_fp32.tsv and read
by select_variant / bench.py.

    python tools/tune_sweep.py --out gpurun_out/tunedb_b200_fp32.tsv [--batches 1,5,20] [--reps 5]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1611_06945_b200 import corpus, tuner  # noqa: E402
from paper_1611_06945_b200.frontend import with_fused  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--batches", default="1,5,20")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--rows", default=None, help="comma list of corpus rows (default all)")
    ap.add_argument("--merge", default=None, help="existing DB to merge into")
    ap.add_argument("--prec", type=int, default=0, help="0 fp32-exact, 1 bf16 mode")
    ap.add_argument("--all-out", default=None, help="CSV of every valid candidate (sig, variant, params, ns, ctas)")
    ap.add_argument("--nets", default="alexnet,nin,googlenet_3a",
                    help="also tune the conv nodes of these network files (data/nets) at the same batches")
    args = ap.parse_args()
    db = tuner.load_db(args.merge) if args.merge and os.path.exists(args.merge) else tuner.TuneDB()
    rows = None if args.rows is None else {int(r) for r in args.rows.split(",")}
    t_all = time.time()
    cand = [] if args.all_out else None
    for row, op in corpus.sweep_ops([int(b) for b in args.batches.split(",")]):
        if rows is not None and row not in rows:
            continue
        g = with_fused(op.graph(), "conv", "relu")
        node = g.node("conv")
        t0 = time.time()
        rec = tuner.sweep(node, g.edges, reps=args.reps, warmup=2, prec=args.prec, record_all=cand)
        db.add(rec)
        print(f"row{row:02d} N={op.batch:2d} {rec.op_signature:42s} {rec.variant:11s} {rec.params.to_string():60s} "
              f"{rec.cost / 1e3:9.2f} us  {op.flops_computed / rec.cost / 1e3:7.1f} TFLOP/s  err={rec.max_rel_err:.2e}  "
              f"({time.time() - t0:.1f}s)", flush=True)
        tuner.save_db(db, args.out)
    if args.nets and rows is None:
        from paper_1611_06945_b200 import graphopt
        from paper_1611_06945_b200.frontend import KIND_CONV, infer_shapes, parse_net
        from paper_1611_06945_b200.ndarray import DimsSpec

        nets = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1611_06945_b200", "data", "nets")
        for net in args.nets.split(","):
            text = open(os.path.join(nets, f"{net}.net")).read()
            for b in [int(b) for b in args.batches.split(",")]:
                g = parse_net(text)
                d = g.edges["data"]
                g = graphopt.fuse_activations(infer_shapes(g, DimsSpec.row_major(d.names, (b,) + d.sizes[1:])))
                for node in g.nodes:
                    if node.kind != KIND_CONV or tuner.op_signature(node, g.edges) in db.records:
                        continue
                    rec = tuner.sweep(node, g.edges, reps=args.reps, warmup=2, prec=args.prec, record_all=cand)
                    db.add(rec)
                    print(f"{net} N={b:2d} {rec.op_signature:42s} {rec.variant:11s} {rec.params.to_string():60s} "
                          f"{rec.cost / 1e3:9.2f} us", flush=True)
                tuner.save_db(db, args.out)
    if cand is not None:
        with open(args.all_out, "w") as fh:
            fh.write("signature,variant,params,ns,ctas\n")
            for sig, vname, ps, ns, ctas in cand:
                fh.write(f"{sig},{vname},\"{ps}\",{ns},{ctas}\n")
    print(f"tuned {len(db.records)} signatures in {time.time() - t_all:.0f}s -> {args.out}")


if __name__ == "__main__":
    main()
