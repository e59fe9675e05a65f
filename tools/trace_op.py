#!/usr/bin/env python
"""Phase trace of CTA 0 of the TMA conv kernel (debug):
    python tools/trace_op.py --row 6 --batch 1 --params 'MNt=4:4,...,tm=1' [--variant conv_umma]"""
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
ap.add_argument("--flags", type=int, default=1, help="trace flags: 1 trace, |2 hi*hi only, |4 no split")
a = ap.parse_args()
op = corpus.corpus(a.batch)[a.row]
g = with_fused(op.graph(), "conv", "relu")
node = g.node("conv")
v, p = VARIANTS[a.variant], TuneParams.from_string(a.params)
inputs = runner.node_test_inputs(node, g.edges, "trace")
x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
o = runner.ConvOp(v.generate(node, g.edges, p), x, w, b)
L = backend.lib()
for _ in range(3):
    o.launch()
torch.cuda.synchronize()
L.b2c_debug_trace_enable(a.flags)
buf = (ctypes.c_longlong * 256)()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for rep in range(2):
    ctypes.memset(buf, 0, ctypes.sizeof(buf))
    flush.zero_()
    torch.cuda.synchronize()
    o.launch()
    torch.cuda.synchronize()
    L.b2c_debug_trace_read(buf)
    t0 = buf[0]
    names = {0: "entry", 1: "setup", 2: "split_end", 3: "tid0_pdl", 4: "drains_done", 5: "mma_last_commit", 6: "epi_done", 7: "exit", 8: "ld_early", 9: "ld_pdl", 10: "ld2_top", 11: "ld2_empty", 12: "ld2_expect", 13: "ld2_pixtma", 14: "ld_after_wait"}
    print(f"--- row{a.row} N={a.batch} {p.to_string()} rep{rep} (clk rel. entry)")
    print("  " + "  ".join(f"{names[i]}={buf[i] - t0}" for i in sorted(names) if buf[i]))
    def row(name, base):
        print(f"  {name:11s}" + " ".join(f"{buf[base + i] - t0:6d}" for i in range(32) if buf[base + i]))
    row("tma_issue", 176)
    row("split_raw", 16)
    row("split_done", 48)
    print("  drain/epi  " + " ".join(f"{buf[208 + 2 * i] - t0}/{buf[209 + 2 * i] - t0}" for i in range(24) if buf[208 + 2 * i]))
    row("mma_raw", 80)
    row("mma_split", 112)
    row("mma_commit", 144)
ms_dbg = o.time_ms(warmup=2, reps=10, l2_flush=True)
print(f"time with flags {a.flags}: {ms_dbg * 1e3:.2f} us")
L.b2c_debug_trace_enable(0)
ms = o.time_ms(warmup=2, reps=10, l2_flush=True)
print(f"time {ms * 1e3:.2f} us")
