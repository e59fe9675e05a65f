#!/usr/bin/env python
"""Whole-network forward on the B200: AlexNet / NiN /
GoogLeNet-3a from paper_1611_06945_b200/data/nets at N = 1/5/20, every node one
libb2conv launch, the pass captured in one CUDA graph and timed with CUDA
events (warm, inputs resident).  Prints one JSON line per (net, batch) with the
per-kind time split (from an event-instrumented replay of the same launches).
    python tools/net_bench.py [--nets alexnet,nin,googlenet_3a] [--batches 1,5,20] [--db PATH]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1611_06945_b200 import runner, tuner  # noqa: E402
from paper_1611_06945_b200.frontend import infer_shapes, parse_net  # noqa: E402
from paper_1611_06945_b200.ndarray import DimsSpec  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--nets", default="alexnet,nin,googlenet_3a")
ap.add_argument("--batches", default="1,5,20")
ap.add_argument("--db", default=os.path.join(ROOT, "paper_1611_06945_b200", "data", "tunedb_b200_fp32.tsv"))
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
db = tuner.load_db(a.db) if a.db and os.path.exists(a.db) else None

for net in a.nets.split(","):
    text = open(os.path.join(ROOT, "paper_1611_06945_b200", "data", "nets", f"{net}.net")).read()
    for n in [int(b) for b in a.batches.split(",")]:
        g = parse_net(text)
        d = g.edges["data"]
        g = infer_shapes(g, DimsSpec.row_major(d.names, (n,) + d.sizes[1:]))
        plan = runner.plan_graph(g, db=db)
        ex = runner.GraphExec(plan, seed=f"netbench:{net}")
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                ex.launch(st.cuda_stream)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            with torch.cuda.graph(graph, stream=st):
                ex.launch(st.cuda_stream)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(a.reps):
                graph.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        # per-node split (events between launches: serialises PDL overlap, so the sum exceeds ms)
        split = {}
        with torch.cuda.stream(st):
            evs = []
            for name in plan.order:
                b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                b0.record(st)
                ex.launch_node(name, st.cuda_stream)
                b1.record(st)
                evs.append((name, b0, b1))
        torch.cuda.synchronize()
        for name, b0, b1 in evs:
            v = plan.choices[name][0]
            split[v] = split.get(v, 0.0) + b0.elapsed_time(b1)
        flops = ex.flops
        print(json.dumps({"net": net, "batch": n, "nodes": len(plan.order), "ms": round(ms, 4),
                          "conv_tflops": round(flops / ms / 1e9, 2), "images_per_s": round(n / ms * 1e3, 1),
                          "flops": flops, "split_ms_by_variant": {k: round(v, 4) for k, v in sorted(split.items())}}),
              flush=True)
