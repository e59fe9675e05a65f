"""Command-line driver: bench, tune, run, emit (cuclgen/cli.py on the B200).

    python -m paper_1611_06945_b200.cli bench [--corpus CSV] [--batch N] [--db TSV] [--out CSV] [--flops-only]
    python -m paper_1611_06945_b200.cli tune  [--corpus CSV | --net FILE] [--batch N] --out TSV
    python -m paper_1611_06945_b200.cli run   --net FILE [--batch N] [--db TSV] [--check] [--no-fuse] [--seed S]
    python -m paper_1611_06945_b200.cli emit  --net FILE [--db TSV] [--out DIR]

Same subcommands, report columns (cli.py:23), corpus gate (cli.py:31-51) and
exit codes (cli.py:25-28: 0 ok, 2 validation failure, 3 parse error, 4
internal error) as the reference.  What changes is where the work runs:

* ``bench`` runs each op's chosen kernel at its TRUE shape on the B200 and
  reports the CUDA-event median as ``cost`` (objective ``wall``); its
  ``oracle`` column is the device-side check the tuner uses — the output
  against the exact-order ``conv_simple`` kernel (variants.py:223-276) at the
  reference tolerance (oracle.py:31-38, 124-137) — instead of a downscaled
  twin on the simulator (cli.py:86-101).  The CPU oracle is test-only here.
* ``tune`` is ``tuner.sweep`` (on-device timing) per distinct signature.
* ``run`` is ``runner.run_graph`` on the B200; ``--check`` validates every
  conv node against ``conv_simple`` on the device (pool / ReLU / conversion
  are exact ops, pinned bit-exactly by tests/test_net_gpu.py).
* ``emit``: the reference writes CUCL source text per node (cli.py:164-194);
  here kernels are compiled ahead of time, so ``emit`` writes the chosen
  kernel instantiation (variant, tune string, launch descriptor) per node.
"""

from __future__ import annotations

import argparse
import csv
import os
import sys

from . import corpus as corpus_mod
from . import runner, tuner
from .errors import CuclgenError
from .frontend import KIND_CONV, NetSyntaxError, infer_shapes, parse_net
from .ndarray import DimsSpec
from .variants import STATIC, VARIANTS, TuneParams, select_variant

REPORT_COLUMNS = "signature,variant,params,cost,objective,oracle,max_rel_err"
EXIT_OK, EXIT_VALIDATION, EXIT_PARSE, EXIT_INTERNAL = 0, 2, 3, 4


def _ops(args):
    ops = corpus_mod.load_corpus(args.corpus or corpus_mod.shipped_corpus_path())
    return [op.with_batch(args.batch) for op in ops] if args.batch else ops


def _net(args):
    with open(args.net, encoding="utf-8") as fh:
        g = parse_net(fh.read())
    if args.batch and "data" in g.edges and g.edges["data"] is not None:
        d = g.edges["data"]
        g = infer_shapes(g, DimsSpec.row_major(d.names, (args.batch,) + tuple(d.sizes[1:])))
    return g


def _write(args, rows):
    if args.out and args.out != "-":
        with open(args.out, "w", newline="") as fh:
            csv.writer(fh, lineterminator="\n").writerows(rows)
    else:
        csv.writer(sys.stdout, lineterminator="\n").writerows(rows)


def device_check(node, edges, x, w, b, y, seed="check", prec: int = 0):
    """(ok, max_rel_err) of a conv output ``y`` against the exact-order
    conv_simple kernel on the same device operands, at the tolerance of the
    precision mode the output was computed in (``TuneParams.prec``)."""
    import torch

    ref = runner.ConvOp(VARIANTS["conv_simple"].generate(node, edges, TuneParams()), x, w, b)
    ref.launch()
    torch.cuda.synchronize()
    tol = tuner.tolerance_for(runner.conv_reduction_terms(node, edges), prec)
    return tuner.device_compare(y, ref.y, tol)


def cmd_bench(args) -> int:
    ops = _ops(args)
    problems = corpus_mod.corpus_gate(ops)
    if problems:
        for p in problems:
            print(f"corpus gate: {p}", file=sys.stderr)
        return EXIT_VALIDATION
    db = tuner.load_db(args.db) if args.db else None
    rows, failures = [REPORT_COLUMNS.split(",")], 0
    for op in ops:
        g = op.graph()
        node = g.node("conv")
        if args.relu:
            from .frontend import with_fused

            g = with_fused(g, "conv", "relu")
            node = g.node("conv")
        sig = tuner.op_signature(node, g.edges)
        variant, params = select_variant(node, g.edges, db)
        if args.flops_only:
            rows.append([sig, variant.name, params.to_string(), str(op.flops_computed), "flops", "skipped", ""])
            continue
        inputs = runner.node_test_inputs(node, g.edges, f"bench:{sig}")
        x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
        op_dev = runner.ConvOp(variant.generate(node, g.edges, params, STATIC), x, w, b)
        op_dev.launch()
        ok, err = device_check(node, g.edges, x, w, b, op_dev.y, prec=params.prec)
        ms = op_dev.time_ms(warmup=2, reps=5, l2_flush=True)
        failures += 0 if ok else 1
        rows.append([sig, variant.name, params.to_string(), f"{ms * 1e6:.0f}", tuner.WALL, "pass" if ok else "fail",
                     f"{err:.3e}"])
    _write(args, rows)
    return EXIT_VALIDATION if failures else EXIT_OK


def _tune_nodes(args):
    if args.net:
        g = _net(args)
        return [(n, g.edges) for n in g.nodes if n.kind == KIND_CONV]
    out = []
    for op in _ops(args):
        g = op.graph()
        out.append((g.node("conv"), g.edges))
    return out


def cmd_tune(args) -> int:
    out = args.out or args.db
    if not out:
        print("no output path given (--out or --db)", file=sys.stderr)
        return EXIT_INTERNAL
    db = tuner.TuneDB()
    for node, edges in _tune_nodes(args):
        sig = tuner.op_signature(node, edges)
        if sig in db.records:
            continue
        rec = tuner.sweep(node, edges, objective=tuner.WALL, jobs=args.jobs)
        db.add(rec)
        print(f"{sig}\t{rec.variant}\t{rec.params.to_string()}\t{rec.cost}")
    tuner.save_db(db, out)
    return EXIT_OK


def cmd_run(args) -> int:
    if not args.net:
        print("--net is required", file=sys.stderr)
        return EXIT_PARSE
    g = _net(args)
    db = tuner.load_db(args.db) if args.db else None

    def check(node, edges, inputs, got):
        if node.kind != KIND_CONV:
            return None
        x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
        prec = select_variant(node, edges, db)[1].prec  # the mode run_graph's plan chose for this node
        return device_check(node, edges, x, w, b, runner.to_device(got), prec=prec)

    res = runner.run_graph(g, seed=args.seed, db=db, check=check if args.check else None, fuse=not args.no_fuse)
    for nr in res.node_runs:
        print(f"node {nr.name}: variant={nr.variant} params={nr.params.to_string()} wall_ns={nr.report.wall_ns}")
    for edge, digest in sorted(res.checksums.items()):
        print(f"sink {edge}: {digest}")
    failed = False
    for name, r in res.oracle_checks.items():
        if r is None:
            print(f"check {name}: exact op (not re-checked)")
            continue
        ok, err = r
        failed |= not ok
        print(f"check {name}: " + ("pass" if ok else f"FAIL (rel err {err:.3e})"))
    return EXIT_VALIDATION if failed else EXIT_OK


def _desc_dict(desc) -> dict:
    if isinstance(desc, int):
        return {"elems": desc}
    if hasattr(desc, "out_sizes"):
        n = desc.ndim
        return {"ndim": n, "out_sizes": list(desc.out_sizes)[:n], "src_sizes": list(desc.src_sizes)[:n],
                "src_strides": list(desc.src_strides)[:n]}
    return {f: getattr(desc, f) for f, _ in desc._fields_}


def cmd_emit(args) -> int:
    if not args.net:
        print("--net is required", file=sys.stderr)
        return EXIT_PARSE
    g = _net(args)
    db = tuner.load_db(args.db) if args.db else None
    plan = runner.plan_graph(g, db=db)
    os.makedirs(args.out or ".", exist_ok=True)
    for name in plan.order:
        node = plan.graph.node(name)
        vname, params = plan.choices[name]
        inst = plan.insts[name]
        sig = tuner.op_signature(node, plan.graph.edges)
        desc = _desc_dict(inst.desc)
        if hasattr(inst, "tune"):
            desc["tune"] = {f: getattr(inst.tune, f) for f, _ in inst.tune._fields_}
        fname = f"{sig.replace(':', '_')}__{vname}.plan"
        with open(os.path.join(args.out or ".", fname), "w") as fh:
            fh.write(f"signature {sig}\nvariant {vname}\nparams {params.to_string()}\nkernel {inst.name}\n"
                     f"desc {desc}\n")
        print(f"emitted {fname}")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="b200conv", description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="command", required=True)
    for name, fn in (("bench", cmd_bench), ("tune", cmd_tune), ("run", cmd_run), ("emit", cmd_emit)):
        p = sub.add_parser(name)
        p.add_argument("--net", help="network description file")
        p.add_argument("--corpus", help="benchmark corpus CSV (defaults to the shipped corpus)")
        p.add_argument("--batch", type=int, default=0, help="override the image count (corpus rows / network input)")
        p.add_argument("--db", help="tuning database path")
        p.add_argument("--objective", choices=["model", "wall"], default="wall")
        p.add_argument("--check", action="store_true", help="run: validate conv nodes on device")
        p.add_argument("--no-fuse", action="store_true", help="disable activation fusion")
        p.add_argument("--relu", action="store_true", help="bench: fused ReLU on every op")
        p.add_argument("--flops-only", action="store_true", help="bench: verify corpus only, skip kernel runs")
        p.add_argument("--jobs", type=int, default=1)
        p.add_argument("--seed", default="0")
        p.add_argument("--out", help="output file or directory")
        p.set_defaults(fn=fn)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if args.objective == "model":
        print("error: objective 'model' is the simulator's counter model; the B200 path times on device ('wall')",
              file=sys.stderr)
        return EXIT_INTERNAL
    try:
        return args.fn(args)
    except (NetSyntaxError, corpus_mod.CorpusParseError, tuner.FormatVersionMismatch) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_PARSE
    except (CuclgenError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INTERNAL


if __name__ == "__main__":
    sys.exit(main())
