#!/usr/bin/env python
"""Per-launch device time of one op replayed K times inside one CUDA graph
(no L2 flush: small ops stay L2-resident), for a list of debug flag settings.
    python tools/op_overhead.py --row 6 --batch 1 --params '...' [--flags 0,16]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1611_06945_b200 import backend, corpus, runner  # noqa: E402
from paper_1611_06945_b200.frontend import with_fused  # noqa: E402
from paper_1611_06945_b200.variants import VARIANTS, TuneParams  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--row", type=int, required=True)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--variant", default="conv_umma")
ap.add_argument("--params", required=True)
ap.add_argument("--flags", default="0")
ap.add_argument("--k", type=int, default=50)
a = ap.parse_args()
op = corpus.corpus(a.batch)[a.row]
g = with_fused(op.graph(), "conv", "relu")
node = g.node("conv")
inputs = runner.node_test_inputs(node, g.edges, "ovh")
x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
o = runner.ConvOp(VARIANTS[a.variant].generate(node, g.edges, TuneParams.from_string(a.params)), x, w, b)
L = backend.lib()
st = torch.cuda.Stream()
for fl in [int(f) for f in a.flags.split(",")]:
    L.b2c_debug_trace_enable(fl)
    o.launch()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        with torch.cuda.graph(graph, stream=st):
            for _ in range(a.k):
                o.launch(st.cuda_stream)
    torch.cuda.synchronize()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(5):
            graph.replay()
        e1.record(st)
    torch.cuda.synchronize()
    print(f"row{a.row} N={a.batch} {a.variant} {a.params} flags={fl}: {e0.elapsed_time(e1) * 1e3 / (5 * a.k):.2f} us/launch (graph, warm L2)")
L.b2c_debug_trace_enable(0)
