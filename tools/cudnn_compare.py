#!/usr/bin/env python
"""Informational comparator (not on the product path): the same 129-op sweep
through torch.nn.functional.conv2d + relu (cuDNN), fp32 with TF32 disabled and,
separately, with TF32 allowed, timed as one CUDA graph per batch on warm
inputs the way bench.py times its own graph.
    python tools/cudnn_compare.py [--batches 1,5,20] [--out per_op.csv]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_1611_06945_b200 import corpus  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,5,20")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--out", default=None)
a = ap.parse_args()
torch.backends.cudnn.benchmark = True


def graph_ms(fns, reps):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for _ in range(3):
            for f in fns:
                f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for f in fns:
            f()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rows = []
for tf32 in (False, True):
    torch.backends.cudnn.allow_tf32 = tf32
    total_ms, total_fl = 0.0, 0
    for n in [int(b) for b in a.batches.split(",")]:
        fns, fl_n = [], 0
        for i, op in enumerate(corpus.corpus(n)):
            c, h, w = op.in_chans, op.in_y, op.in_x
            x = torch.rand(n, c, h, w, device="cuda")
            wt = torch.rand(op.out_chans, c, op.ksz, op.ksz, device="cuda")
            b = torch.rand(op.out_chans, device="cuda")
            s, p = op.stride, op.pad

            def f(x=x, wt=wt, b=b, s=s, p=p):
                return F.relu(F.conv2d(x, wt, b, stride=s, padding=p))

            fns.append(f)
            fl = op.flops_computed
            fl_n += fl
            if a.out and tf32 is False:
                ms = graph_ms([f], a.reps * 4)
                rows.append((i, n, f"k{op.ksz}s{op.stride}p{op.pad}oc{op.out_chans}in{n}x{c}x{h}x{w}", ms, fl / ms / 1e9))
        ms = graph_ms(fns, a.reps)
        total_ms += ms
        total_fl += fl_n
        print(f"cudnn tf32={tf32} N={n}: {ms:.4f} ms  {fl_n / ms / 1e9:.2f} TFLOP/s")
    print(f"cudnn tf32={tf32} sweep: {total_ms:.4f} ms/step  {total_fl / total_ms / 1e9:.2f} TFLOP/s")
if a.out:
    with open(a.out, "w") as fh:
        fh.write("row,batch,sig,ms,tflops\n")
        for r in rows:
            fh.write(",".join(str(v) for v in r) + "\n")
