#!/usr/bin/env python
"""Benchmark: conv TFLOP/s + runtime per op over the AlexNet / NiN / GoogLeNet conv sweep at N = 1/5/20.

One *step* = one pass of the hot path over the metric's workload: every op
of the 43-op corpus (cuclgen/corpus.py:28-72) at batch 1, 5
and 20 — 129 convolutions, all with fused bias + ReLU — each on the variant
and tile the shipped on-device-tuned TuneDB selects (select_variant, the
reference's variants.py:840-856 contract).  Synthetic inputs follow the
reference recipe (seed "bench:<op_signature>", U[0.1, 1) fp32).

* ``value``   TFLOP/s of the whole step, operands resident in HBM, the step
  replayed as CUDA graphs, CUDA events on the launching stream, max over
  ranks.  The 129 ops are independent (run_kernel over disjoint
  buffers may run in parallel), so the graph runs them on ``--streams``
  concurrent branches: small ops fill the SMs big ones leave idle.  The
  step's working set (~0.6 GB) is > L2 (126 MB).
* ``per_op``  every op's own runtime (the metric's "runtime per op"): the
  same launches replayed one at a time with an event between ops.
* ``e2e``     the same metric through the public host-buffer call
  (b2c_conv_fwd_host: pinned H2D of x/w/bias, kernel, D2H of y per op).
* ``roofline`` the dominant kernel (largest per-op time).
* ``cpu_baseline`` the reference's own CPU path (cuclgen.oracle.ref_conv from
  the unmodified reference in baseline/_ref; the test-only oracle port when
  that is absent) on a bounded sample of the sweep, all host cores.

Multi-GPU (``--gpus N``; re-launches itself under torch.distributed.run when
WORLD_SIZE is unset): default ``--mode shard`` = north_star config 5 over
the whole sweep (strong scaling): every unit's batch is cut into per-rank
image slabs (20 over 8 ranks -> 3,3,3,3,2,2,2,2; smaller batches by single
images, LPT), and every slab is gathered to rank 0 over NCCL point-to-point,
overlapped with the following compute.  ``value`` is gather-inclusive;
``multi_gpu.compute_only`` excludes the gather.  ``--mode weak``: every rank
runs the whole sweep on its own images (no collective on the data path).

``--impl reference`` times the reference's CPU implementation of the path
(cuclgen.oracle.ref_conv, the float64 direct conv every reference test
compares against) over all 129 ops per step on the host cores of rank 0 and
prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv TFLOP/s + runtime per op, AlexNet/NiN/GoogLeNet sweep at N=1/5/20"
WORKLOAD = "alexnet+nin+googlenet conv sweep: 43 corpus ops x N in {1,5,20}, fused bias+ReLU, fp32"
REF_SITE = os.path.join(ROOT, "baseline", "_ref", "site")

E2E_STREAMS = int(os.environ.get("B2C_E2E_STREAMS", "4"))

# SURVEY.md §8(d) configs 1-3 (corpus rows)
CONFIG1 = (34, 1)
CONFIG2_ROWS = (34, 42, 38, 40, 37)
CONFIG3_ROWS = (2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 14, 18, 19)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--batches", default="1,5,20")
    ap.add_argument("--prec", choices=("fp32", "bf16", "fp8"), default="fp32",
                    help="fp32: fp32-exact (3xTF32 / FFMA, the headline); bf16: bf16 operands, fp32 accumulate "
                         "(separately stated tolerance rel 4e-3); fp8: e4m3 operands, fp32 accumulate (rel 0.13, the per-product rounding bound)")
    ap.add_argument("--db", default=None,
                    help="latency TuneDB for the per-op runtimes (default: shipped B200 DB of the precision)")
    ap.add_argument("--sweep-db", default=None,
                    help="TuneDB for the concurrent step (default: the shipped *_sweep DB: per op the candidate "
                         "minimising time x (CTAs/148)^0.5 within 3x of the fastest, tools/pick_db.py)")
    ap.add_argument("--heuristic", action="store_true", help="ignore the TuneDB, use select_variant's heuristic")
    ap.add_argument("--streams", type=int, default=int(os.environ.get("B2C_BENCH_STREAMS", "16")),
                    help="concurrent graph branches the independent ops are spread over (1 = serial)")
    ap.add_argument("--mode", choices=("shard", "weak"), default="shard",
                    help="multi-GPU: shard = each unit's batch split across ranks + NCCL gather to rank 0 "
                         "(strong, north_star config 5); weak = every rank runs the sweep on its own images")
    ap.add_argument("--no-gather", action="store_true", help="shard mode: skip the output gather")
    ap.add_argument("--groups", choices=("auto", "one", "batch"), default="auto",
                    help="CUDA graphs per step: one (all ops concurrent), batch (one per batch size; the gather of "
                         "a group overlaps the next group); auto = batch when gathering, else one")
    ap.add_argument("--per-op-out", default=None, help="write the per-op CSV here")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget (s)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--debug-flags", type=int, default=0,
                    help="library debug flags (measurement experiments only; results are then not valid bench lines)")
    return ap.parse_args(argv)


# ----------------------------------------------------------------------------- helpers

def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    # /opt/skills/guides/B200_PROFILING.md fallbacks
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_cores() -> int:
    threads = os.environ.get("OPENBLAS_NUM_THREADS") or os.environ.get("OMP_NUM_THREADS")
    return int(threads) if threads else len(os.sched_getaffinity(0))


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    ~2 ms during the timed region (nvidia-smi as a fallback)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4,
               "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None
            self.max_mhz = None

    def _sample(self):
        if self._nvml is not None:
            p = self._nvml
            sm = float(p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM))
            try:
                mask = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                mask = p.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
            self.rows.append((sm, int(mask)))
            return
        out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,"
                              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        if out.returncode == 0 and out.stdout.strip():
            v = [s.strip() for s in out.stdout.strip().split(",")]
            bits = (0x8, 0x40, 0x20, 0x4)
            mask = sum(b for b, s in zip(bits, v[2:6]) if s == "Active")
            self.max_mhz = float(v[1]) if v[1].replace(".", "").isdigit() else self.max_mhz
            self.rows.append((float(v[0]), mask))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(0.002 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.rows:
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({n for _, m in self.rows for n, bit in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def measure_tf32_peak(dev, reps: int = 10) -> float:
    """Dense TF32 throughput of a cuBLAS 8192^3 matmul (2*N^3 / best time), the
    denominator of the 3xTF32 ceiling."""
    import torch

    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        c = torch.empty(n, n, device=dev)
        for _ in range(3):
            torch.matmul(a, b, out=c)
        best = float("inf")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(reps):
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b, c
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def measure_pcie(dev, nbytes: int = 1 << 28, reps: int = 3) -> dict:
    """Pinned-host copy bandwidth (GB/s): H2D alone, D2H alone, and each direction
    while both run at once -- the denominator of the e2e copy bound."""
    import torch

    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_out = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    cur = torch.cuda.current_stream(dev)
    out = {}
    for name in ("h2d", "d2h", "both"):
        best = float("inf")
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record(cur)
            s_h2d.wait_event(e0)
            s_d2h.wait_event(e0)
            if name != "d2h":
                with torch.cuda.stream(s_h2d):
                    d_in.copy_(h_in, non_blocking=True)
            if name != "h2d":
                with torch.cuda.stream(s_d2h):
                    h_out.copy_(d_out, non_blocking=True)
            cur.wait_stream(s_h2d)
            cur.wait_stream(s_d2h)
            e1.record(cur)
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e1))
        out[name + "_gbs"] = round(nbytes / (best * 1e-3) / 1e9, 2)
    del h_in, h_out, d_in, d_out
    return out


def build_sweep(batches, db, heuristic, prec=0):
    """(row, BenchOp, node, edges, variant, params) for every unit of the sweep."""
    from paper_1611_06945_b200 import corpus
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.variants import select_variant

    out = []
    for row, op in corpus.sweep_ops(batches):
        g = with_fused(op.graph(), "conv", "relu")
        node = g.node("conv")
        # a record of the requested precision mode, else the heuristic re-targeted to it
        v, params = select_variant(node, g.edges, None if heuristic else db, prec=prec)
        out.append((row, op, node, g.edges, v, params))
    return out


def make_inputs(op, node, edges, image_seed_suffix=""):
    """Reference synthetic operands (runner.node_test_inputs recipe, seed
    "bench:<signature>:<edge>")."""
    from paper_1611_06945_b200 import runner, tuner

    sig = tuner.op_signature(node, edges)
    data = runner.noise(edges["data"].names, edges["data"].sizes, runner.seed_for(f"bench:{sig}:data{image_seed_suffix}"))
    f = runner.noise(edges["conv_filts"].names, edges["conv_filts"].sizes, runner.seed_for(f"bench:{sig}:conv_filts"))
    b = runner.noise(edges["conv_bias"].names, edges["conv_bias"].sizes, runner.seed_for(f"bench:{sig}:conv_bias"))
    return data.to_np(), f.to_np(), b.to_np()


# ----------------------------------------------------------------------------- CPU reference path

def load_reference():
    """The unmodified reference (cuclgen) from baseline/_ref (baseline/fetch_ref.sh), or None."""
    if not os.path.isdir(os.path.join(REF_SITE, "cuclgen")):
        return None
    if REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    try:
        import cuclgen.corpus
        import cuclgen.oracle
        import cuclgen.runner
        import cuclgen.tuner  # noqa: F401

        return cuclgen
    except Exception:
        return None


class CpuSweep:
    """The sweep on the host: the reference's own ``runner.node_reference`` ->
    ``oracle.ref_conv`` (oracle.py:69-99, float64 numpy/OpenBLAS) on the
    reference's own synthetic inputs (``runner.node_test_inputs``, seed
    "bench:<signature>"), or — without baseline/_ref — the oracle port
    (oracle/conv_ref.py, test infrastructure) on the same recipe."""

    def __init__(self, batches):
        self.ref = load_reference()
        self.units = []
        if self.ref is not None:
            from dataclasses import replace

            R = self.ref
            ops = R.corpus.corpus()
            for b in batches:
                for row, op in enumerate(ops):
                    g = replace(op, batch=b).graph()
                    g.nodes = [replace(nd, fused_activation="relu") if nd.name == "conv" else nd for nd in g.nodes]
                    node = g.node("conv")
                    sig = R.tuner.op_signature(node, g.edges)
                    out = g.edges[node.outputs[0]]
                    flops = 2 * op.ksz ** 2 * op.in_chans * op.out_chans * b * out.size_of("y") * out.size_of("x")
                    self.units.append((row, b, node, g.edges, sig, flops))
            self.kind = "reference"
            self.what = "cuclgen.runner.node_reference -> cuclgen.oracle.ref_conv (unmodified reference, baseline/_ref)"
        else:
            from paper_1611_06945_b200 import corpus

            for row, op in corpus.sweep_ops(batches):
                self.units.append((row, op.batch, None, op, None, op.flops_computed))
            self.kind = "port"
            self.what = "oracle/conv_ref.ref_conv (numpy float64 port; baseline/_ref absent)"
        self._inputs = {}

    def inputs(self, i):
        if i not in self._inputs:
            row, b, node, edges, sig, _ = self.units[i]
            if self.kind == "reference":
                self._inputs[i] = self.ref.runner.node_test_inputs(node, edges, f"bench:{sig}")
            else:
                import numpy as np

                op = edges
                rng = np.random.default_rng(row * 100 + b)
                x = rng.uniform(0.1, 1.0, (op.batch, op.in_chans, op.in_y, op.in_x)).astype(np.float32)
                f = rng.uniform(0.1, 1.0, (op.out_chans, op.in_chans, op.ksz, op.ksz)).astype(np.float32)
                bb = rng.uniform(0.1, 1.0, op.out_chans).astype(np.float32)
                self._inputs[i] = (x, f, bb)
        return self._inputs[i]

    def run(self, i) -> float:
        """Seconds of one unit's CPU conv (inputs generated beforehand, untimed)."""
        inp = self.inputs(i)
        row, b, node, edges, sig, _ = self.units[i]
        if self.kind == "reference":
            t0 = time.perf_counter()
            self.ref.runner.node_reference(node, edges, inp)
            return time.perf_counter() - t0
        from oracle import conv_ref

        op = edges
        t0 = time.perf_counter()
        conv_ref.ref_conv(*inp, op.stride, op.pad, relu=True)
        return time.perf_counter() - t0

    def sample(self, budget_s: float):
        """Units in sweep order until ~budget_s of conv time: (flops, seconds, n)."""
        flops, secs, n = 0, 0.0, 0
        for i in range(len(self.units)):
            if secs > budget_s:
                break
            secs += self.run(i)
            flops += self.units[i][5]
            n += 1
            self._inputs.pop(i, None)
        return flops, secs, n


def cpu_baseline(batches, budget_s):
    """The reference's CPU path on a bounded sample of the sweep (units in
    sweep order), all host cores; plus a one-thread sample of a third of the
    budget."""
    cs = CpuSweep(batches)
    flops, secs, n = cs.sample(budget_s)
    out = {"value": round(flops / secs / 1e12, 6), "unit": "TFLOP/s", "cores": host_cores(), "kind": cs.kind,
           "sample": f"first {n} of {len(cs.units)} sweep units in sweep order (N={batches[0]} first): {cs.what}",
           "seconds": round(secs, 2), "flops": flops, "cpu_model": cpu_model()}
    try:
        from threadpoolctl import threadpool_limits

        with threadpool_limits(limits=1):
            f1, s1, n1 = cs.sample(budget_s / 3)
        out["one_thread"] = {"value": round(f1 / s1 / 1e12, 6), "units": n1, "seconds": round(s1, 2)}
    except Exception as e:  # threadpoolctl missing: report why
        out["one_thread"] = {"unavailable": str(e)[:80]}
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path over the whole sweep, every step."""
    if rank != 0:
        return
    batches = [int(b) for b in args.batches.split(",")]
    cs = CpuSweep(batches)
    n = len(cs.units)
    flops_step = sum(u[5] for u in cs.units)
    for i in range(n):  # the reference's synthetic inputs, generated once (untimed)
        cs.inputs(i)
    per_unit = [0.0] * n
    steps = []
    for s in range(args.warmup + args.steps):
        t = [cs.run(i) for i in range(n)]
        if s >= args.warmup:
            steps.append(sum(t))
            for i in range(n):
                per_unit[i] += t[i] / args.steps
    secs = statistics.median(steps)
    v = flops_step / secs / 1e12
    one = None
    try:
        from threadpoolctl import threadpool_limits

        n1 = sum(1 for u in cs.units if u[1] == cs.units[0][1])  # the first batch group (N=1 units)
        with threadpool_limits(limits=1):
            t1 = [cs.run(i) for i in range(n1)]
        one = {"value": round(sum(u[5] for u in cs.units[:n1]) / sum(t1) / 1e12, 6),
               "units": n1, "seconds": round(sum(t1), 2)}
    except Exception as e:
        one = {"unavailable": str(e)[:80]}
    by_batch = {}
    for i, u in enumerate(cs.units):
        e = by_batch.setdefault(u[1], [0.0, 0])
        e[0] += per_unit[i]
        e[1] += u[5]
    sample = f"all {n} sweep units per step: {cs.what}"
    line = {"metric": METRIC, "value": round(v, 6), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * secs, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD, "global_batch": "1,5,20", "parallelism": "host cores",
                       "ops_per_step": n, "flops_per_step": flops_step, "sample": sample,
                       "per_batch_s": {str(k): round(e[0], 3) for k, e in sorted(by_batch.items())}},
            "cpu_baseline": {"value": round(v, 6), "unit": "TFLOP/s", "cores": host_cores(), "kind": cs.kind,
                             "sample": sample, "cpu_model": cpu_model(), "one_thread": one},
            "e2e": {"value": round(v, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm

def capture(graph_ops, streams):
    """One CUDA graph launching ``graph_ops`` [(ConvOp, est. ms)] over
    len(streams) concurrent branches: ops are dealt longest-first to the
    least-loaded branch (LPT), so the branches finish together."""
    import torch

    g = torch.cuda.CUDAGraph()
    s0 = streams[0]
    with torch.cuda.stream(s0):
        with torch.cuda.graph(g, stream=s0):
            if len(streams) == 1:
                for o, _ in graph_ops:
                    o.launch(s0.cuda_stream)
            else:
                fork = torch.cuda.Event()
                fork.record(s0)
                for s in streams[1:]:
                    s.wait_event(fork)
                loads = [0.0] * len(streams)
                for i in sorted(range(len(graph_ops)), key=lambda i: (-graph_ops[i][1], i)):
                    k = min(range(len(streams)), key=lambda j: (loads[j], j))
                    loads[k] += graph_ops[i][1]
                    graph_ops[i][0].launch(streams[k].cuda_stream)
                for s in streams[1:]:
                    j = torch.cuda.Event()
                    j.record(s)
                    s0.wait_event(j)
    return g


def run_ours(args, rank, world, local_rank, one_gpu_test=False):
    import torch
    import torch.distributed as dist

    from paper_1611_06945_b200 import backend as be
    from paper_1611_06945_b200 import runner, shard, tuner
    from paper_1611_06945_b200.backend import conv_bytes, conv_flops
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.variants import select_variant

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if args.debug_flags:
        be.lib().b2c_debug_trace_enable(args.debug_flags & ~1)  # never the (CTA-0 trace) bit
    batches = [int(b) for b in args.batches.split(",")]
    prec = {"fp32": 0, "bf16": 1, "fp8": 2}[args.prec]
    db_path = args.db or tuner.shipped_db_path(args.prec)
    db = tuner.load_db(db_path) if (os.path.exists(db_path) and not args.heuristic) else None
    sdb_path = args.sweep_db or tuner.shipped_db_path(args.prec + "_sweep")
    sdb = tuner.load_db(sdb_path) if (os.path.exists(sdb_path) and not args.heuristic) else db
    if sdb is db:
        sdb_path = db_path
    sweep = build_sweep(batches, sdb, args.heuristic, prec)  # the step's kernel choices
    shard_mode = world > 1 and args.mode == "shard"
    gather = shard_mode and not args.no_gather

    # ---- this rank's work items
    def est_cost(u, count):
        row, op, node, edges, v, params = sweep[u]
        return op.flops_computed * count / op.batch  # time ~ flops

    if shard_mode:
        items = shard.plan_sweep([s[1].batch for s in sweep], world, est_cost)
    else:
        items = [shard.WorkItem(u, rank, 0, s[1].batch) for u, s in enumerate(sweep)]
    full_out = {}  # rank 0, shard mode: every unit's full output (slabs land in place)
    if shard_mode and rank == 0:
        for u, (row, op, node, edges, v, params) in enumerate(sweep):
            osz = edges[node.outputs[0]].sizes
            full_out[u] = torch.empty(tuple(osz), dtype=torch.float32, device=dev)
    # ops: per-op runtimes (latency DB: one op at a time); sops: the step (sweep DB, concurrent);
    # the same ConvOp where both DBs pick the same kernel and tile
    ops, sops, sw_est, hosts, rows = [], [], [], [], []
    for it in items:
        if it.rank != rank:
            continue
        row, op, node, edges, v, params = sweep[it.unit]
        # weak mode: every rank its own images; shard mode: the slab of the unit's images
        x, f, b = make_inputs(op, node, edges, "" if shard_mode or rank == 0 else f":r{rank}")
        if shard_mode and it.count != op.batch:  # a slab: the DBs' choices for the slab's batch size
            op = op.with_batch(it.count)
            g = with_fused(op.graph(), "conv", "relu")
            node, edges = g.node("conv"), g.edges
            v, params = select_variant(node, edges, None if args.heuristic else sdb, prec=prec)
            x = x[it.first: it.first + it.count]
        vl, pl = select_variant(node, edges, None if args.heuristic else db, prec=prec)
        sig = tuner.op_signature(node, edges)
        plan = v.generate(node, edges, params)
        dx, df, db_ = (torch.from_numpy(a.copy()).to(dev) for a in (x, f, b))
        y = full_out[it.unit][it.first: it.first + it.count] if it.unit in full_out else None
        sop = runner.ConvOp(plan, dx, df, db_, y=y)
        same = vl.name == v.name and pl.to_string() == params.to_string()
        ops.append(sop if same else runner.ConvOp(vl.generate(node, edges, pl), dx, df, db_))
        sops.append(sop)
        rec = sdb.records.get(sig) if sdb is not None else None
        sw_est.append(rec.cost * 1e-6 if rec is not None else op.flops_computed / 1e11)  # ms, for the LPT branches
        if not args.no_e2e:
            hosts.append(runner.HostRun.create(plan, x, f, b, device=dev))
        rows.append((row, op, vl.name, pl, sig, it, v.name, params))
    torch.cuda.synchronize()
    pack_ms = sum(o.prepare_ms() for o in sops)  # one-time filter packs (cached per filter tensor)
    for o, so in zip(ops, sops):
        if o is not so:
            o.prepare()
    flops_mine = sum(conv_flops(o.plan.desc) for o in sops)
    launches_mine = sum(int(be.lib().b2c_conv_launches(be.ctypes.byref(o.plan.desc), be.ctypes.byref(o.tune)))
                        for o in sops)
    n_same = sum(1 for o, so in zip(ops, sops) if o is so)
    tf32 = measure_tf32_peak(dev) if rank == 0 else None

    # ---- per-op isolated timing (the metric's "runtime per op"): serial graph, event between ops
    n = len(ops)
    main = torch.cuda.Stream(device=dev)
    for o in ops + sops:  # warm every kernel once (smem attributes, module load) outside capture
        o.launch()
    torch.cuda.synchronize()
    per_op = [0.0] * n
    if n:
        evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(n + 1)]
        graph_ev = torch.cuda.CUDAGraph()
        with torch.cuda.stream(main):
            with torch.cuda.graph(graph_ev, stream=main):
                evs[0].record(main)
                for i, o in enumerate(ops):
                    o.launch(main.cuda_stream)
                    evs[i + 1].record(main)
        for rep in range(args.warmup + args.steps):
            graph_ev.replay()
            torch.cuda.synchronize()
            if rep >= args.warmup:
                for i in range(n):
                    per_op[i] += evs[i].elapsed_time(evs[i + 1]) / args.steps

    # ---- per-op back-to-back: each op launched R times in one CUDA graph (what a launch costs
    # when the next one queues behind it: no event nodes between launches, ~4 us each; the
    # inputs stay L2-resident between launches except fc6's 151 MB of weights)
    R_B2B = 8
    per_op_b2b = [0.0] * n
    for i, o in enumerate(ops):
        gb2b = torch.cuda.CUDAGraph()
        with torch.cuda.stream(main):
            with torch.cuda.graph(gb2b, stream=main):
                for _ in range(R_B2B):
                    o.launch(main.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gb2b.replay()
        best = float("inf")
        for _ in range(3):
            with torch.cuda.stream(main):
                e0.record(main)
                gb2b.replay()
                e1.record(main)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / R_B2B)
        per_op_b2b[i] = best
        del gb2b
    torch.cuda.synchronize()

    # ---- the timed step: one group per batch size (the same groups on every rank), each one
    # CUDA graph over concurrent branches; shard mode: after a group, its slabs go to rank 0
    # (NCCL p2p on NCCL's stream, overlapping the next group's compute)
    nstreams = max(1, args.streams)
    streams = [main] + [torch.cuda.Stream(device=dev) for _ in range(nstreams - 1)]
    per_batch = args.groups == "batch" or (args.groups == "auto" and gather)
    group_of = (lambda u: sweep[u][1].batch) if per_batch else (lambda u: 0)
    groups = []
    for gb in sorted({group_of(u) for u in range(len(sweep))}):
        gitems = [it for it in items if group_of(it.unit) == gb]
        idx = [i for i, r in enumerate(rows) if group_of(r[5].unit) == gb]
        local = {gitems.index(rows[i][5]): sops[i].y for i in idx}
        graph = capture([(sops[i], sw_est[i]) for i in idx], streams) if idx else None
        groups.append((gb, graph, gitems, local))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    def one_step(ev_groups=None):
        works = []
        for gi, (gb, graph, gitems, local) in enumerate(groups):
            if graph is not None:
                graph.replay()
            if ev_groups is not None:
                ev_groups[gi].record(main)
            if gather:
                works += shard.gather_to_root(gitems, local, full_out, rank, stage_cpu=one_gpu_test)
        return works

    with torch.cuda.stream(main):
        for _ in range(args.warmup):
            for w in one_step():
                w.wait()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t_c = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t_g = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_groups = [[torch.cuda.Event(enable_timing=True) for _ in groups] for _ in range(args.steps)]
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        with torch.cuda.stream(main):
            t0.record(main)
            for s in range(args.steps):
                works = one_step(ev_groups[s])
                t_c[s].record(main)
                for w in works:
                    w.wait()  # the gather lands before the next step rewrites the buffers
                t_g[s].record(main)
        torch.cuda.synchronize()
    ms_step = t0.elapsed_time(t_g[-1]) / args.steps
    starts = [t0] + t_g[:-1]
    compute_ms = statistics.mean(starts[s].elapsed_time(t_c[s]) for s in range(args.steps))
    group_ms = [statistics.mean((starts[s] if gi == 0 else ev_groups[s][gi - 1]).elapsed_time(ev_groups[s][gi])
                                for s in range(args.steps)) for gi in range(len(groups))]
    if world > 1:
        tt = torch.tensor([ms_step, compute_ms, *group_ms], dtype=torch.float64, device=dev)
        tt = tt.cpu() if one_gpu_test else tt
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_step, compute_ms, group_ms = float(tt[0]), float(tt[1]), [float(v) for v in tt[2:]]
    flops_all = flops_mine
    if world > 1:
        ft = torch.tensor([float(flops_mine)], dtype=torch.float64, device=dev)
        ft = ft.cpu() if one_gpu_test else ft
        dist.all_reduce(ft, op=dist.ReduceOp.SUM)
        flops_all = float(ft.item())
    value = flops_all / (ms_step * 1e-3) / 1e12

    # ---- e2e through the host-buffer C call (each rank: its own slabs, host in, host out)
    e2e = None
    if hosts or (world > 1 and not args.no_e2e):
        side = [torch.cuda.Stream(device=dev) for _ in range(E2E_STREAMS)]
        # the ops are independent: interleave the most input-heavy with the most output-heavy ones
        # so that the H2D and D2H copy engines stay busy together (profiles/r2am/e2e_probe.log)
        by_ratio = sorted(hosts, key=lambda h: h.d2h_bytes / max(1, h.h2d_bytes))
        e2e_order = [by_ratio[(j // 2) if j % 2 == 0 else len(by_ratio) - 1 - j // 2] for j in range(len(by_ratio))]
        for h in hosts:
            h.run(main.cuda_stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ksteps = max(1, min(args.steps, 5))
        with torch.cuda.stream(main):
            e0.record(main)
            for s in side:
                s.wait_event(e0)
            for _ in range(ksteps):
                for i, h in enumerate(e2e_order):
                    h.run(side[i % E2E_STREAMS].cuda_stream)
            for s in side:
                main.wait_stream(s)
            e1.record(main)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / ksteps
        if world > 1:
            tt = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            tt = tt.cpu() if one_gpu_test else tt
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        h2d_b, d2h_b = sum(h.h2d_bytes for h in hosts), sum(h.d2h_bytes for h in hosts)
        pcie = measure_pcie(dev)
        # copy bound: both directions stream concurrently at the measured duplex rate
        copy_ms = max(h2d_b / (pcie["both_gbs"] * 1e9), d2h_b / (pcie["both_gbs"] * 1e9)) * 1e3
        e2e = {"value": round(flops_all / (e_ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s", "ms_per_step": round(e_ms, 3),
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b, "steps": ksteps,
               "pcie_measured": pcie, "copy_bound_ms": round(copy_ms, 3),
               "frac_of_copy_bound": round(copy_ms / e_ms, 4),
               "path": f"b2c_conv_fwd_host per op (pinned H2D x/w/bias + filter pack + kernel + D2H y), "
                       f"ops round-robin on {E2E_STREAMS} streams, input-heavy and output-heavy ops interleaved" + (" (bytes: rank 0's share)" if world > 1 else "")}

    if rank != 0:
        return
    peaks = load_peaks()
    tf32_mode = tf32 / 3.0  # 3xTF32: three TF32 MMA passes per useful product
    # fp8: the nominal dense fp8 rate is 2x bf16 (no measured fp8 peak in MEASURED_PEAKS.json)
    mode_peak = {0: tf32_mode, 1: peaks["bf16_tflops"], 2: 2.0 * peaks["bf16_tflops"]}[prec]

    def frac_of_roof(fl_i, by_i, ms):
        t_roof = max(fl_i / (mode_peak * 1e12), by_i / (peaks["hbm_gbs"] * 1e9))
        return t_roof / (ms * 1e-3)

    # ---- roofline of the dominant kernel (largest isolated per-op time)
    roof = None
    if n:
        dom = max(range(n), key=lambda i: per_op[i])
        d = ops[dom]
        fl, by, t_ms = conv_flops(d.plan.desc), conv_bytes(d.plan.desc), per_op[dom]
        ridge = mode_peak * 1e12 / (peaks["hbm_gbs"] * 1e9)
        if fl / by >= ridge:
            achieved = fl / (t_ms * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": round(achieved, 3), "peak": peaks["bf16_tflops"],
                    "unit": "TFLOP/s", "frac": round(achieved / peaks["bf16_tflops"], 4),
                    "mode_peak": round(mode_peak, 1), "frac_of_mode_peak": round(achieved / mode_peak, 4),
                    "mode_peak_note": ("bf16 mode: measured bf16 dense peak" if prec == 1 else
                                       "fp8 mode: 2 x the measured bf16 dense peak (nominal fp8 rate)" if prec == 2 else
                                       "fp32-exact 3xTF32 ceiling = TF32 dense measured in this run "
                                       "(cuBLAS 8192^3) / 3 passes")}
        else:
            achieved = by / (t_ms * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": round(achieved / peaks["hbm_gbs"], 4)}
        r_row, r_op, r_var, r_par, r_sig = rows[dom][:5]
        roof.update({"traffic": None, "peak_source": peaks["source"], "tf32_measured_tflops": round(tf32, 1),
                     "kernel": f"{r_var} [{r_par.to_string()}]", "op": r_sig, "corpus_row": r_row,
                     "share_of_step": round(t_ms / sum(per_op), 4), "launch_ms": round(t_ms, 4),
                     "algorithmic_flops": fl, "algorithmic_bytes": by})
        traffic_file = os.path.join(ROOT, "profiles", "dominant_traffic.json")
        if os.path.exists(traffic_file):
            with open(traffic_file) as fh:
                tj = json.load(fh)
            if tj.get("op") == r_sig and tj.get("kernel_params") == r_par.to_string():
                roof["traffic"] = tj.get("traffic_bytes")
                roof["traffic_source"] = tj.get("source")

    # ---- per-op table (rank 0's items), configs 1-3 and 5
    per_rows = []
    for i, (row, op, vname, params, sig, it) in enumerate(r[:6] for r in rows):
        fl_i, by_i = conv_flops(ops[i].plan.desc), conv_bytes(ops[i].plan.desc)
        per_rows.append([row, op.batch, round(per_op[i] * 1e3, 2), round(fl_i / per_op[i] / 1e9, 2),
                         round(frac_of_roof(fl_i, by_i, per_op[i]), 4), round(per_op_b2b[i] * 1e3, 2)])
    if args.per_op_out:
        with open(args.per_op_out, "w") as fh:
            fh.write("row,batch,signature,variant,params,ms,tflops,gbs,flops,bytes,frac_roofline,sweep_variant,sweep_params\n")
            for i, (row, op, vname, params, sig, it, sv, sp) in enumerate(rows):
                fl_i, by_i = conv_flops(ops[i].plan.desc), conv_bytes(ops[i].plan.desc)
                fh.write(f"{row},{op.batch},{sig},{vname},\"{params.to_string()}\",{per_op[i]:.5f},"
                         f"{fl_i / per_op[i] / 1e9:.3f},{by_i / per_op[i] / 1e6:.1f},{fl_i},{by_i},"
                         f"{frac_of_roof(fl_i, by_i, per_op[i]):.4f},{sv},\"{sp.to_string()}\"\n")

    def subset(pred):
        idx = [i for i, r in enumerate(rows) if pred(r[0], sweep[r[5].unit][1].batch)]
        if not idx:
            return None
        ms = sum(per_op[i] for i in idx)
        fl_s = sum(conv_flops(ops[i].plan.desc) for i in idx)
        roof_ms = sum(frac_of_roof(conv_flops(ops[i].plan.desc), conv_bytes(ops[i].plan.desc), per_op[i]) * per_op[i]
                      for i in idx)
        return {"ops": len(idx), "us": round(ms * 1e3, 2), "tflops": round(fl_s / ms / 1e9, 2),
                "frac_roofline": round(roof_ms / ms, 4)}

    configs = {"config1_alexnet_conv1_n1": subset(lambda r, b: (r, b) == CONFIG1),
               "config2_alexnet_conv1_5": {str(b): subset(lambda r, bb, b=b: r in CONFIG2_ROWS and bb == b)
                                           for b in batches},
               "config3_googlenet_1x1_n20": subset(lambda r, b: r in CONFIG3_ROWS and b == 20),
               "config5_all_n20": subset(lambda r, b: b == 20)}

    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_baseline(batches, args.cpu_seconds)
    by_batch = {}
    for i, (row, op, vname, params, sig, it) in enumerate(r[:6] for r in rows):
        e = by_batch.setdefault(sweep[it.unit][1].batch, [0.0, 0, 0.0])
        e[0] += per_op[i]
        e[1] += conv_flops(ops[i].plan.desc)
        e[2] += per_op_b2b[i]
    roof_ms_mine = sum(frac_of_roof(conv_flops(o.plan.desc), conv_bytes(o.plan.desc), per_op[i]) * per_op[i]
                       for i, o in enumerate(ops))
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong" if shard_mode else "weak",
        "vs_baseline": None, "dtype": args.prec, "data": "synthetic",
        "config": {"workload": WORKLOAD if not prec else WORKLOAD.replace(
                       ", fp32", ", bf16 operands / fp32 accumulate" if prec == 1 else ", e4m3 operands / fp32 accumulate"),
                   "global_batch": ",".join(str(b if shard_mode else b * world) for b in batches),
                   "sharding": ("per-unit image slabs over ranks (20 over 8: 3,3,3,3,2,2,2,2; smaller batches "
                                "by single images, LPT) - strong" if shard_mode
                                else ("N images per rank (weak)" if world > 1 else "none (1 GPU)")),
                   "output_gather": ("every slab to rank 0 by NCCL p2p after its batch group, overlapping the "
                                     "next group; inside the timed step" if gather else "none"),
                   "ops_per_step": len(sweep), "launches_rank0": n, "flops_per_step": int(flops_all),
                   "parallelism": f"batch-shard x{world}" if world > 1 else "1 GPU",
                   "variant_source": "heuristic" if db is None else
                   {"per_op": os.path.relpath(db_path, ROOT), "step": os.path.relpath(sdb_path, ROOT),
                    "ops_with_same_choice": n_same},
                   "l2": "working set ~0.6 GB > 126 MB L2 (no explicit flush)",
                   "schedule": (f"{len(groups)} CUDA graph(s) per step" + (" (one per batch size)" if per_batch else "")
                                + f", the ops of a graph on {nstreams} concurrent branches (LPT by per-op time)"),
                   "filter_pack_ms_once": round(pack_ms, 3),
                   "group_ms": {("batch " + str(g[0]) if per_batch else "all"): round(ms, 4) for g, ms in zip(groups, group_ms)},
                   "per_batch_ms_isolated": {str(k): round(v[0], 4) for k, v in sorted(by_batch.items())},
                   "per_batch_tflops_isolated": {str(k): round(v[1] / v[0] / 1e9, 2) for k, v in sorted(by_batch.items())},
                   "per_batch_ms_back_to_back": {str(k): round(v[2], 4) for k, v in sorted(by_batch.items())},
                   "per_op_timing": ("us: isolated (serial graph, an event node after every op: ~4 us of event "
                                     "overhead included); us_b2b: the op launched 8x back to back in one graph "
                                     "(launch gaps included, inputs L2-warm except fc6)"),
                   "serial_ms_per_step_rank0": round(sum(per_op), 4),
                   "roofline_ms_rank0": round(roof_ms_mine, 4),
                   "frac_roofline_step": round(roof_ms_mine / ms_step, 4) if world == 1 else None,
                   **configs},
        "roofline": roof,
        "per_op": {"cols": ["row", "n", "us", "tflops", "frac_roofline", "us_b2b"], "rows": per_rows},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_mine * args.steps,
        "clocks": clocks.summary(),
    }
    if world > 1:
        line["multi_gpu"] = {"mode": args.mode, "gather": gather,
                             "compute_only_ms": round(compute_ms, 4),
                             "compute_only_tflops": round(flops_all / (compute_ms * 1e-3) / 1e12, 3),
                             "gather_inclusive_ms": round(ms_step, 4),
                             "gather_inclusive_tflops": round(value, 3),
                             "note": "max over ranks; compute_only excludes waiting for the gather; "
                                     "gpu_launches, per_op and e2e bytes are rank 0's"}
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (rank 0 prints the line)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # Test hook for the N > 1 control flow on a one-GPU box: every rank on cuda:0,
    # collectives over gloo (NCCL refuses two ranks on one GPU).  Never set by the driver.
    one_gpu_test = os.environ.get("B2C_BENCH_ONE_GPU_TEST") == "1"
    if one_gpu_test:
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if not one_gpu_test and torch.cuda.device_count() < world:
            raise SystemExit(f"bench: {world} ranks but only {torch.cuda.device_count()} visible GPUs")
        torch.cuda.set_device(local_rank)
        if one_gpu_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank, one_gpu_test)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
