"""e2e probe (GPU): raw pinned PCIe bandwidth (H2D, D2H, both at once) and the
host-buffer sweep (b2c_conv_fwd_host per op) at several stream counts and op
orders, to see how close the e2e step gets to its copy bound.

    python tools/e2e_probe.py [--streams 4,8,16,32] [--steps 3]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1611_06945_b200 import runner, tuner  # noqa: E402
from paper_1611_06945_b200.backend import conv_flops  # noqa: E402


def copy_bw(dev, nbytes=1 << 29, reps=5):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    out = {}
    for name in ("h2d", "d2h", "both"):
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            s1.wait_event(e0)
            s2.wait_event(e0)
            if name in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name + "_gbs"] = round(nbytes / (best * 1e-3) / 1e9, 2)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", default="4,8,16,32")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    print(json.dumps({"pcie": copy_bw(dev)}), flush=True)
    db = tuner.load_db(os.path.join(ROOT, "paper_1611_06945_b200/data/tunedb_b200_fp32.tsv"))
    sweep = bench.build_sweep((1, 5, 20), db, False, prec=0)
    hosts, flops = [], 0
    for row, op, node, edges, v, params in sweep:
        x, f, b = bench.make_inputs(op, node, edges)
        plan = v.generate(node, edges, params)
        hosts.append(runner.HostRun.create(plan, x, f, b, device=dev))
        flops += conv_flops(plan.desc)
    h2d = sum(h.h2d_bytes for h in hosts)
    d2h = sum(h.d2h_bytes for h in hosts)
    for h in hosts:
        h.run()
    torch.cuda.synchronize()
    orders = {"sweep": list(range(len(hosts))),
              "bytes_desc": sorted(range(len(hosts)), key=lambda i: -hosts[i].h2d_bytes)}
    # alternate input-heavy and output-heavy ops so both copy directions stay busy
    ratio = sorted(range(len(hosts)), key=lambda i: hosts[i].d2h_bytes / max(1, hosts[i].h2d_bytes))
    alt = []
    lo, hi = 0, len(ratio) - 1
    while lo <= hi:
        alt.append(ratio[lo]); lo += 1
        if lo <= hi:
            alt.append(ratio[hi]); hi -= 1
    orders["alternate"] = alt
    main_s = torch.cuda.current_stream()
    for ns in [int(s) for s in a.streams.split(",")]:
        side = [torch.cuda.Stream(dev) for _ in range(ns)]
        for oname, order in orders.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(main_s)
            for s in side:
                s.wait_event(e0)
            for _ in range(a.steps):
                for j, i in enumerate(order):
                    hosts[i].run(side[j % ns].cuda_stream)
            for s in side:
                main_s.wait_stream(s)
            e1.record(main_s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            print(json.dumps({"streams": ns, "order": oname, "ms": round(ms, 3),
                              "tflops": round(flops / (ms * 1e-3) / 1e12, 3),
                              "h2d_gbs": round(h2d / (ms * 1e-3) / 1e9, 2),
                              "d2h_gbs": round(d2h / (ms * 1e-3) / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    main()
