#!/usr/bin/env python
"""Where a small op's per-launch time goes (measurement tool, GPU box): one op
replayed K times inside one CUDA graph, alone / alternating with a tiny torch
kernel / with an event record between launches (the bench's per-op graph),
against the kernel's own entry->exit span from the phase trace.
    python tools/launch_floor.py --row 3 --batch 1 --variant conv_1x1 --params 'BN=32,sk=4,tm=3'"""
import argparse
import ctypes
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
ap.add_argument("--k", type=int, default=50)
a = ap.parse_args()
op = corpus.corpus(a.batch)[a.row]
g = with_fused(op.graph(), "conv", "relu")
node = g.node("conv")
inputs = runner.node_test_inputs(node, g.edges, "floor")
x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
p = TuneParams.from_string("MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1," + a.params)
o = runner.ConvOp(VARIANTS[a.variant].generate(node, g.edges, p), x, w, b)
tiny = torch.zeros(1024, device="cuda")
st = torch.cuda.Stream()
o.launch()
torch.cuda.synchronize()


def timed(body, label):
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        with torch.cuda.graph(graph, stream=st):
            for _ in range(a.k):
                body()
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
    print(f"  {label:44s} {e0.elapsed_time(e1) * 1e3 / (5 * a.k):7.2f} us per iteration", flush=True)


print(f"row{a.row} N={a.batch} {a.variant} {a.params}")
timed(lambda: o.launch(st.cuda_stream), "op x K (graph)")
timed(lambda: tiny.add_(1.0), "tiny torch kernel x K")
timed(lambda: (o.launch(st.cuda_stream), tiny.add_(1.0)), "op + tiny torch kernel")
ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(a.k)]
it = iter(range(10 ** 9))


def with_event():
    o.launch(st.cuda_stream)
    ev[next(it) % a.k].record(st)


timed(with_event, "op + event record (bench per-op graph)")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
timed(lambda: (flush.add_(1.0), o.launch(st.cuda_stream)), "256 MB write + op (cold L2)")
timed(lambda: flush.add_(1.0), "256 MB write alone")
L = backend.lib()
buf = (ctypes.c_longlong * 256)()
L.b2c_debug_trace_enable(1)
o.launch()
torch.cuda.synchronize()
L.b2c_debug_trace_read(buf)
L.b2c_debug_trace_enable(0)
print(f"  CTA 0 entry->exit span: {(buf[7] - buf[0]) / 1.9e3:.2f} us at 1.9 GHz "
      f"(setup {(buf[1] - buf[0]) / 1.9e3:.2f} us, loader after early loads {(buf[8] - buf[0]) / 1.9e3:.2f}, "
      f"after pdl_wait {(buf[9] - buf[0]) / 1.9e3:.2f}, first TMA {(buf[176] - buf[0]) / 1.9e3:.2f})")
