#!/usr/bin/env python
"""One small launch of every kernel family in libb2conv, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck on every kernel
family; the reference's analogue is its strict permuted-thread-order engine,
cuclgen/backend.py:1038-1087, and the race tests of tests/test_runner.py:38-57).

    compute-sanitizer --tool memcheck python tools/sanitize_ops.py [--quick]

Every launch is also checked against the exact-order conv_simple kernel, so a
sanitizer run doubles as a parity run at these shapes.  Exit status 1 on a
mismatch."""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1611_06945_b200 import backend, runner, tuner  # noqa: E402
from paper_1611_06945_b200.frontend import ConvParams, conv_graph, with_fused  # noqa: E402
from paper_1611_06945_b200.ndarray import DimsSpec  # noqa: E402
from paper_1611_06945_b200.variants import VARIANTS, TuneParams  # noqa: E402

P = "MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,"
# (label, (b, ic, h, w), (ksz, stride, pad, oc), variant, params)
CASES = [
    ("k_simple", (2, 5, 9, 9), (3, 1, 1, 7), "conv_simple", "MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"),
    ("k_tiled", (2, 8, 10, 10), (3, 2, 1, 16), "conv_tiled", "MNt=4:4,MNb=8:8,Kb=8,vw=4,lf=1,li=1"),
    ("k_umma gather", (2, 32, 10, 10), (3, 1, 1, 40), "conv_umma", P + "BN=64,sk=1,sw=0,dr=0"),
    ("k_umma gather swap split", (1, 36, 8, 8), (3, 1, 1, 140), "conv_umma", P + "BN=32,sk=2,sw=1,dr=0"),
    ("k_tconv MODE0 im2col", (2, 64, 12, 12), (3, 1, 1, 96), "conv_umma", P + "BN=96,sk=1,sw=0,dr=0,tm=1"),
    ("k_tconv MODE0 split-K", (1, 64, 12, 12), (3, 1, 1, 64), "conv_umma", P + "BN=64,sk=3,sw=0,dr=0,tm=1"),
    ("k_tconv MODE0 stream-K", (2, 64, 12, 12), (5, 1, 2, 128), "conv_umma", P + "BN=128,sk=0,sw=0,dr=0,tm=1"),
    ("k_tconv MODE0 swap", (1, 32, 9, 9), (3, 1, 1, 130), "conv_umma", P + "BN=64,sk=1,sw=1,dr=0,tm=1"),
    ("k_tconv MODE0 2 CTA/SM", (2, 32, 12, 12), (3, 1, 1, 64), "conv_umma", P + "BN=64,sk=1,sw=0,dr=0,tm=1,oc=2"),
    ("k_tconv MODE0 CTA pair", (2, 32, 12, 12), (3, 1, 1, 64), "conv_umma", P + "BN=64,sk=1,sw=0,dr=0,tm=1,cl=2"),
    ("k_tconv MODE2 1x1 2-D", (2, 64, 10, 10), (1, 1, 0, 48), "conv_1x1", P + "BN=64,sk=1,sw=0,dr=0,tm=2"),
    ("k_tconv MODE5 1x1 NCHW", (2, 64, 12, 12), (1, 1, 0, 48), "conv_1x1", P + "BN=64,sk=2,sw=0,dr=0,tm=3"),
    ("k_tconv MODE6 kxk NCHW", (2, 32, 12, 16), (3, 1, 1, 64), "conv_umma", P + "BN=64,sk=1,sw=0,dr=0,tm=4"),
    ("k_tconv MODE4 first layer", (1, 3, 35, 35), (11, 4, 0, 32), "conv_umma", P + "BN=32,sk=1,sw=0,dr=0,tm=1"),
    ("k_tconv MODE3 first layer 8-tap", (1, 3, 20, 20), (7, 2, 3, 32), "conv_umma", P + "BN=32,sk=1,sw=0,dr=0,tm=2"),
    ("k_tconv MODE1 fc", (2, 16, 4, 4), (4, 1, 0, 96), "conv_fc", P + "BN=32,sk=2,sw=1,dr=0,tm=1"),
    ("k_tconv bf16", (2, 64, 12, 12), (3, 1, 1, 64), "conv_umma", P + "BN=64,sk=1,sw=0,dr=0,tm=1,pr=1"),
    ("k_tconv bf16 1x1 NCHW", (2, 64, 12, 12), (1, 1, 0, 64), "conv_1x1", P + "BN=64,sk=1,sw=0,dr=0,tm=3,pr=1"),
    ("k_fc_stream", (2, 16, 4, 4), (4, 1, 0, 64), "conv_fc_stream", "MNt=1:4,MNb=4:1,Kb=1,vw=1,lf=1,li=1"),
    ("k_fc_smem", (3, 16, 4, 4), (4, 1, 0, 64), "conv_fc_stream", "MNt=1:2,MNb=4:1,Kb=2,vw=1,lf=1,li=1"),
    ("k_fc_bulk", (3, 16, 8, 8), (8, 1, 0, 72), "conv_fc_stream", "MNt=1:1,MNb=8:1,Kb=3,vw=1,lf=1,li=1"),
    ("k_tconv MODE1 fc BN=16", (5, 16, 4, 4), (4, 1, 0, 160), "conv_fc", P + "BN=16,sk=2,sw=1,dr=0,tm=1,oc=2"),
    ("k_tconv MODE0 2-SM pair", (2, 32, 12, 12), (3, 1, 1, 128), "conv_umma", P + "BN=128,sk=1,sw=0,dr=0,tm=1,cl=3"),
    ("k_tconv MODE0 2-SM pair stream-K", (2, 32, 12, 12), (3, 1, 1, 96), "conv_umma", P + "BN=96,sk=0,sw=0,dr=0,tm=1,cl=3"),
    ("k_tconv split-K cluster", (1, 64, 12, 12), (3, 1, 1, 64), "conv_umma", P + "BN=64,sk=2,sw=0,dr=0,tm=1,cl=4"),
    ("k_tconv first-layer space-to-depth", (1, 3, 35, 35), (11, 4, 0, 32), "conv_umma", P + "BN=32,sk=1,sw=0,dr=0,tm=6"),
    ("k_tconv bf16 SS", (2, 64, 12, 12), (3, 1, 1, 128), "conv_umma", P + "BN=128,sk=1,sw=0,dr=0,tm=5,pr=1"),
    ("k_tconv bf16 SS pair", (2, 64, 12, 12), (3, 1, 1, 128), "conv_umma", P + "BN=128,sk=1,sw=0,dr=0,tm=5,cl=3,pr=1"),
    ("k_tconv fp8", (2, 64, 12, 12), (3, 1, 1, 64), "conv_umma", P + "BN=64,sk=1,sw=0,dr=0,tm=1,pr=2"),
    ("k_wino + MODE7", (2, 32, 12, 12), (3, 1, 1, 64), "conv_wino", P + "BN=64,sk=1,sw=0,dr=0"),
]


def graph(in_dims, kp, relu=True):
    k, s, p, oc = kp
    g = conv_graph(ConvParams(ksz=k, stride=s, pad=p, out_chans=oc), DimsSpec.row_major(("img", "chan", "y", "x"), in_dims))
    return with_fused(g, "conv", "relu") if relu else g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="only the first case of each kernel template family")
    ap.add_argument("--only", default=None, help="substring of the case labels to run")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    bad = 0
    for label, dims, kp, vname, ps in CASES:
        if a.only and a.only not in label:
            continue
        g = graph(dims, kp)
        node = g.node("conv")
        params = TuneParams.from_string(ps)
        inputs = runner.node_test_inputs(node, g.edges, f"san:{label}", low=-1.0, high=1.0)
        x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
        op = runner.ConvOp(VARIANTS[vname].generate(node, g.edges, params), x, w, b)
        op.launch()
        ref = runner.ConvOp(VARIANTS["conv_simple"].generate(node, g.edges, TuneParams()), x, w, b)
        ref.launch()
        torch.cuda.synchronize()
        k = {0: 1e-5, 1: 8e-3, 2: 0.14}[params.prec]  # the modes' stated signed bounds (fp8: per-product e4m3)
        # sum|x||w| per output by the exact-order kernel itself (no library conv in a sanitizer run)
        gb = graph(dims, kp, relu=False)
        absop = runner.ConvOp(VARIANTS["conv_simple"].generate(gb.node("conv"), gb.edges, TuneParams()), x.abs(),
                              w.abs(), torch.zeros_like(b))
        absop.launch()
        bound = k * absop.y + 1e-6
        err = (op.y - ref.y).abs()
        ok = bool((err <= bound).all())
        bad += 0 if ok else 1
        print(f"{label:34s} {vname:15s} {ps.split(',BN=')[-1]:28s} {'ok' if ok else 'MISMATCH'}", flush=True)
    # whole-network kernels: pool, ReLU, layout conversion
    xs = torch.randn(2, 5, 9, 11, device="cuda")
    y = torch.empty(2, 5, 5, 6, device="cuda")
    backend.pool_max_fwd(backend.PoolDesc(2, 5, 9, 11, 3, 2, 1, 5, 6), xs, y)
    want = torch.nn.functional.max_pool2d(xs, 3, 2, 1)  # torch's own pooling kernel: reads initialised x only
    print(f"{'k_pool_max':34s} {'ok' if torch.equal(y, want) else 'MISMATCH'}")
    bad += 0 if torch.equal(y, want) else 1
    r = torch.empty_like(xs)
    backend.relu_fwd(xs, r)
    print(f"{'k_relu4':34s} {'ok' if torch.equal(r, xs.clamp_min(0)) else 'MISMATCH'}")
    bad += 0 if torch.equal(r, xs.clamp_min(0)) else 1
    d = backend.xpose_desc(("img", "chan", "y", "x"), (2, 5, 9, 11), [495, 99, 11, 1], ("img", "y", "x", "chan"), (2, 9, 11, 8))
    t = torch.empty(2, 9, 11, 8, device="cuda")
    backend.xpose(d, xs, t)
    want = torch.zeros(2, 9, 11, 8, device="cuda")
    want[..., :5] = xs.permute(0, 2, 3, 1)
    print(f"{'k_xpose_tiled':34s} {'ok' if torch.equal(t, want) else 'MISMATCH'}")
    bad += 0 if torch.equal(t, want) else 1
    torch.cuda.synchronize()
    print("sanitize_ops:", "all ok" if not bad else f"{bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
