#!/usr/bin/env python
"""Benchmark: conv TFLOP/s over the AlexNet / NiN / GoogLeNet conv sweep at N = 1/5/20.

One *step* = one pass of the hot path over the metric's workload: every op
of the 43-op corpus (cuclgen/corpus.py:28-72) at batch 1, 5
and 20 — 129 convolutions, all with fused bias + ReLU — each on the variant
and tile the shipped on-device-tuned TuneDB selects (select_variant, the
reference's variants.py:840-856 contract).  Synthetic inputs follow the
reference recipe (seed "bench:<op_signature>", U[0.1, 1) fp32).

* ``value``   TFLOP/s of the whole step, operands resident in HBM, the 129
  launches replayed as one CUDA graph, CUDA events on the launching stream.
  The step's working set (~0.6 GB) is > L2 (126 MB), so every op's operands
  are evicted by the rest of the sweep between its launches.
* ``e2e``     the same metric through the public host-buffer call
  (b2c_conv_fwd_host: pinned H2D of x/w/bias, kernel, D2H of y per op).
* ``roofline`` the dominant kernel (largest share of the step), timed by
  CUDA events recorded inside the same graph.
* ``cpu_baseline`` the CPU oracle (numpy float64 restatement of the
  reference's ref_conv, all host cores) on a bounded sample of the sweep.

Multi-GPU (torchrun): every rank runs the sweep on its own slab of images
(batch sharding, no data-path collective), ``scaling`` = "weak"; value =
all ranks' FLOPs / max-over-ranks time.

``--impl reference`` times the reference's CPU path (the oracle port) on
rank 0 and prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv TFLOP/s + runtime per op, AlexNet/NiN/GoogLeNet sweep at N=1/5/20"
WORKLOAD = "alexnet+nin+googlenet conv sweep: 43 corpus ops x N in {1,5,20}, fused bias+ReLU, fp32"


E2E_STREAMS = int(os.environ.get("B2C_E2E_STREAMS", "4"))


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--batches", default="1,5,20")
    ap.add_argument("--prec", choices=("fp32", "bf16"), default="fp32",
                    help="fp32: fp32-exact (3xTF32 / FFMA, the headline); bf16: bf16 operands, fp32 accumulate "
                         "(separately stated tolerance rel 4e-3)")
    ap.add_argument("--db", default=None, help="TuneDB path (default: shipped B200 fp32 DB if present)")
    ap.add_argument("--heuristic", action="store_true", help="ignore the TuneDB, use select_variant's heuristic")
    ap.add_argument("--per-op-out", default=None, help="write per-op CSV here")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--strong", action="store_true",
                    help="multi-GPU: split each op's batch across ranks (strong scaling) instead of N images per rank")
    ap.add_argument("--gather", action="store_true",
                    help="multi-GPU: all-gather every op's output slabs over NCCL inside the timed step")
    ap.add_argument("--debug-flags", type=int, default=0,
                    help="library debug flags (measurement experiments only; results are then not valid bench lines)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers

def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([v.strip() for v in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.rows)}


def build_sweep(batches, db, heuristic, rank, world=1, strong=False, prec=0):
    """(row, BenchOp, node, edges, variant, params) for every op of the sweep.
    Weak scaling: every rank runs every op on its own N images.  Strong
    scaling: rank r takes its contiguous slab of each op's N images
    (shard.batch_slab); ops whose slab is empty on this rank are skipped."""
    from paper_1611_06945_b200 import corpus
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.shard import batch_slab
    from paper_1611_06945_b200.variants import select_variant

    out = []
    for row, op in corpus.sweep_ops(batches):
        if strong and world > 1:
            n_local = batch_slab(op.batch, world, rank)[1]
            if n_local == 0:
                continue
            op = op.with_batch(n_local)
        g = with_fused(op.graph(), "conv", "relu")
        node = g.node("conv")
        v, params = select_variant(node, g.edges, None if heuristic else db)
        if prec and params.prec != prec:  # bf16 mode: a record of this precision, else the first bf16 candidate
            from dataclasses import replace

            from paper_1611_06945_b200 import tuner

            params = replace(params, prec=prec)
            if v.applies(node, g.edges, params) is not None:
                v, params = tuner.candidates(node, g.edges, prec=prec)[0]
        out.append((row, op, node, g.edges, v, params))
    return out


def make_inputs(op, node, edges, rank):
    """Reference synthetic operands (runner.node_test_inputs recipe); per-rank
    images, shared filters (batch sharding)."""
    from paper_1611_06945_b200 import runner, tuner

    sig = tuner.op_signature(node, edges)
    data = runner.noise(edges["data"].names, edges["data"].sizes, runner.seed_for(f"bench:{sig}:data" + (f":r{rank}" if rank else "")))
    f = runner.noise(edges["conv_filts"].names, edges["conv_filts"].sizes, runner.seed_for(f"bench:{sig}:conv_filts"))
    b = runner.noise(edges["conv_bias"].names, edges["conv_bias"].sizes, runner.seed_for(f"bench:{sig}:conv_bias"))
    return data.to_np(), f.to_np(), b.to_np()


def cpu_baseline(batches, budget_s):
    """Time the CPU oracle (oracle/conv_ref.py, numpy float64, all cores) on a
    bounded sample of the sweep: ops in sweep order until ~budget_s seconds."""
    import numpy as np

    from oracle import conv_ref
    from paper_1611_06945_b200 import corpus

    flops, secs, n = 0, 0.0, 0
    t_start = time.perf_counter()
    for row, op in corpus.sweep_ops(batches):
        if time.perf_counter() - t_start > budget_s:
            break
        x = np.random.default_rng(row).uniform(0.1, 1.0, (op.batch, op.in_chans, op.in_y, op.in_x)).astype(np.float32)
        f = np.random.default_rng(row + 1000).uniform(0.1, 1.0, (op.out_chans, op.in_chans, op.ksz, op.ksz)).astype(np.float32)
        b = np.zeros(op.out_chans, np.float32)
        t0 = time.perf_counter()
        conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=True)
        secs += time.perf_counter() - t0
        flops += op.flops_computed
        n += 1
    threads = os.environ.get("OPENBLAS_NUM_THREADS") or os.environ.get("OMP_NUM_THREADS")
    cores = int(threads) if threads else len(os.sched_getaffinity(0))
    return {"value": round(flops / secs / 1e12, 6), "unit": "TFLOP/s", "cores": cores, "kind": "port",
            "sample": f"first {n} ops of the sweep in sweep order (N={batches[0]} first), oracle/conv_ref.ref_conv float64",
            "seconds": round(secs, 2), "flops": flops}


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    if rank != 0:
        return
    batches = [int(b) for b in args.batches.split(",")]
    vals = []
    per_step_budget = max(2.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(batches, per_step_budget)
        if i >= args.warmup:
            vals.append(cb)
    v = statistics.median(c["value"] for c in vals)
    cb = vals[-1]
    line = {"metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.median(c["seconds"] for c in vals), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD, "global_batch": "1,5,20", "parallelism": "host cores",
                       "sample": cb["sample"]},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cb["cores"], "kind": "port",
                             "sample": cb["sample"]},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1611_06945_b200 import runner, tuner
    from paper_1611_06945_b200.backend import conv_bytes, conv_flops

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if args.debug_flags:
        from paper_1611_06945_b200 import backend as _bk
        _bk.lib().b2c_debug_trace_enable(args.debug_flags & ~1)  # never the (CTA-0 trace) bit
    batches = [int(b) for b in args.batches.split(",")]
    prec = 1 if args.prec == "bf16" else 0
    db_path = args.db or tuner.shipped_db_path(args.prec)
    db = tuner.load_db(db_path) if (os.path.exists(db_path) and not args.heuristic) else None
    sweep = build_sweep(batches, db, args.heuristic, rank, world, args.strong, prec)

    ops, hosts, rows = [], [], []
    for row, op, node, edges, v, params in sweep:
        x, f, b = make_inputs(op, node, edges, rank)
        plan = v.generate(node, edges, params)
        dx, df, db_ = (torch.from_numpy(a).to(dev) for a in (x, f, b))
        ops.append(runner.ConvOp(plan, dx, df, db_))
        if not args.no_e2e:
            hosts.append(runner.HostRun.create(plan, x, f, b, device=dev))
        rows.append((row, op, v.name, params, tuner.op_signature(node, edges)))
    torch.cuda.synchronize()
    pack_ms = sum(o.prepare_ms() for o in ops)  # one-time filter packs (cached per filter tensor)
    flops_step = sum(conv_flops(o.plan.desc) for o in ops)
    from paper_1611_06945_b200 import backend as _be
    launches_per_step = sum(int(_be.lib().b2c_conv_launches(_be.ctypes.byref(o.plan.desc), _be.ctypes.byref(o.tune)))
                            for o in ops)
    stream = torch.cuda.Stream(device=dev)

    # ---- capture the step as one CUDA graph (the timed one: kernels only), and a
    # second copy with an event node between ops for the per-op breakdown
    n = len(ops)
    evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(n + 1)]
    for o in ops:  # warm every kernel once (smem attributes, module load) outside capture
        o.launch()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(graph, stream=stream):
            for o in ops:
                o.launch(stream.cuda_stream)
    graph_ev = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(graph_ev, stream=stream):
            evs[0].record(stream)
            for i, o in enumerate(ops):
                o.launch(stream.cuda_stream)
                evs[i + 1].record(stream)
    torch.cuda.synchronize()

    gather = args.gather and world > 1
    if gather:
        from paper_1611_06945_b200.shard import gather_batch
        if args.strong:
            raise SystemExit("--gather is implemented for weak scaling (every rank holds every op)")
        n_fulls = [world * op.batch for (_, op, _, _, _) in rows]  # all ranks' images of each op
    for _ in range(args.warmup):
        graph.replay()
        if gather:
            with torch.cuda.stream(stream):
                for o, n_full in zip(ops, n_fulls):
                    gather_batch(o.y, n_full)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_op = [0.0] * n
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        with torch.cuda.stream(stream):
            t0.record(stream)
            for _ in range(args.steps):
                graph.replay()
                if gather:
                    for o, n_full in zip(ops, n_fulls):
                        gather_batch(o.y, n_full)
            t1.record(stream)
        torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    # per-op times: the event-instrumented copy of the step, replayed after the timed region
    for _ in range(args.steps):
        graph_ev.replay()
        torch.cuda.synchronize()
        for i in range(n):
            per_op[i] += evs[i].elapsed_time(evs[i + 1]) / args.steps
    ms_step = total_ms / args.steps
    if world > 1:
        tt = torch.tensor([ms_step], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_step = float(tt.item())
    flops_all = world * flops_step
    if world > 1 and args.strong:  # ranks hold different slabs: sum the work actually done
        ft = torch.tensor([float(flops_step)], device=dev, dtype=torch.float64)
        dist.all_reduce(ft, op=dist.ReduceOp.SUM)
        flops_all = float(ft.item())
    value = flops_all / (ms_step * 1e-3) / 1e12

    # ---- e2e through the host-buffer C call
    e2e = None
    if hosts:
        # Independent ops go round-robin over E2E_STREAMS streams, so one op's
        # D2H overlaps the next op's H2D (PCIe is full duplex) and kernels.
        side = [torch.cuda.Stream(device=dev) for _ in range(E2E_STREAMS)]
        for h in hosts:
            h.run(stream.cuda_stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ksteps = max(1, min(args.steps, 5))
        with torch.cuda.stream(stream):
            e0.record(stream)
            for s in side:
                s.wait_event(e0)
            for _ in range(ksteps):
                for i, h in enumerate(hosts):
                    h.run(side[i % E2E_STREAMS].cuda_stream)
            for s in side:
                stream.wait_stream(s)
            e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / ksteps
        if world > 1:
            tt = torch.tensor([e_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        e2e = {"value": round(world * flops_step / (e_ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
               "ms_per_step": round(e_ms, 3),
               "h2d_bytes_per_step": sum(h.h2d_bytes for h in hosts),
               "d2h_bytes_per_step": sum(h.d2h_bytes for h in hosts), "steps": ksteps,
               "path": f"b2c_conv_fwd_host per op (pinned H2D x/w/bias + kernel + D2H y), ops round-robin on {E2E_STREAMS} streams"}

    if rank != 0:
        return
    peaks = load_peaks()
    # ---- roofline of the dominant kernel
    dom = max(range(n), key=lambda i: per_op[i])
    d = ops[dom]
    fl, by, t_ms = conv_flops(d.plan.desc), conv_bytes(d.plan.desc), per_op[dom]
    # 3xTF32: TF32 = bf16/2, three MMA passes; bf16 mode: one kind::f16 pass
    mode_peak = peaks["bf16_tflops"] if prec else peaks["bf16_tflops"] / 2 / 3
    ridge = mode_peak * 1e12 / (peaks["hbm_gbs"] * 1e9)
    tensor_bound = fl / by >= ridge
    if tensor_bound:
        achieved = fl / (t_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": round(achieved, 3), "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": round(achieved / peaks["bf16_tflops"], 4),
                "mode_peak": round(mode_peak, 1), "frac_of_mode_peak": round(achieved / mode_peak, 4),
                "mode_peak_note": ("bf16 mode: measured bf16 dense peak" if prec else
                                   "fp32-exact 3xTF32 ceiling = measured bf16 dense / 2 (TF32 rate) / 3 (passes)")}
    else:
        achieved = by / (t_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4)}
    r_row, r_op, r_var, r_par, r_sig = rows[dom]
    roof.update({"traffic": None, "peak_source": peaks["source"], "kernel": f"{r_var} [{r_par.to_string()}]",
                 "op": r_sig, "corpus_row": r_row, "share_of_step": round(t_ms / sum(per_op), 4),
                 "launch_ms": round(t_ms, 4), "algorithmic_flops": fl, "algorithmic_bytes": by})
    traffic_file = os.path.join(ROOT, "profiles", "dominant_traffic.json")
    if os.path.exists(traffic_file):
        with open(traffic_file) as fh:
            tj = json.load(fh)
        if tj.get("op") == r_sig and tj.get("kernel_params") == r_par.to_string():
            roof["traffic"] = tj.get("traffic_bytes")

    if args.per_op_out:
        with open(args.per_op_out, "w") as fh:
            fh.write("row,batch,signature,variant,params,ms,tflops,gbs,flops,bytes\n")
            for i, (row, op, vname, params, sig) in enumerate(rows):
                fl_i, by_i = conv_flops(ops[i].plan.desc), conv_bytes(ops[i].plan.desc)
                fh.write(f"{row},{op.batch},{sig},{vname},\"{params.to_string()}\",{per_op[i]:.5f},"
                         f"{fl_i / per_op[i] / 1e9:.3f},{by_i / per_op[i] / 1e6:.1f},{fl_i},{by_i}\n")

    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_baseline(batches, args.cpu_seconds)
    by_batch = {}
    for i, (row, op, vname, params, sig) in enumerate(rows):
        e = by_batch.setdefault(op.batch, [0.0, 0])
        e[0] += per_op[i]
        e[1] += conv_flops(ops[i].plan.desc)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "strong" if (args.strong and world > 1) else "weak",
        "vs_baseline": None, "dtype": args.prec, "data": "synthetic",
        "config": {"workload": WORKLOAD if not prec else WORKLOAD.replace(", fp32", ", bf16 operands / fp32 accumulate"),
                   "global_batch": ",".join(str(b if args.strong else b * world) for b in batches),
                   "sharding": "batch slabs per op (strong)" if args.strong else "N images per rank (weak)",
                   "output_gather": "NCCL all_gather of every op's slabs, inside the timed step" if gather else "none",
                   "ops_per_step": n, "flops_per_step_per_gpu": flops_step, "parallelism": f"batch-shard x{world}",
                   "variant_source": "heuristic" if db is None else os.path.relpath(db_path, ROOT),
                   "l2": "working set ~0.6 GB > 126 MB L2 (no explicit flush)",
                   "graph": "one CUDA graph per step (kernels only); per-op times from an event-instrumented copy",
                   "filter_pack_ms_once": round(pack_ms, 3),
                   "per_batch_ms": {str(k): round(v[0], 4) for k, v in sorted(by_batch.items())},
                   "per_batch_tflops": {str(k): round(v[1] / v[0] / 1e9, 2) for k, v in sorted(by_batch.items())}},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # Test hook for the N > 1 control flow on a one-GPU box: every rank on cuda:0,
    # collectives over gloo (NCCL refuses two ranks on one GPU).  Never set by the driver.
    if os.environ.get("B2C_BENCH_ONE_GPU_TEST") == "1":
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if os.environ.get("B2C_BENCH_ONE_GPU_TEST") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
