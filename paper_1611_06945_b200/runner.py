"""Execution harness: run one conv op through libb2conv.

Mirrors the single-op part of cuclgen/runner.py: ``node_test_inputs``
(runner.py:39-45, with the seeded-noise recipe of oracle.py:48-60),
``conv_reduction_terms`` (:66-70) and ``execute_node`` (:73-106) — canonical
NdArrays in, canonical NdArray + CostReport out, output written into a
caller-shaped buffer.  The kernel runs on the B200 through the C ABI; the
CostReport's ``wall_ns`` is the kernel's CUDA-event time.

``ConvOp`` is the device-resident form used by the tuner and the bench: the
operands live in HBM and ``launch()`` issues exactly one kernel on the
current stream (so it can be captured in a CUDA graph).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

from . import backend
from .backend import CostReport
from .errors import CuclgenError
from .frontend import KIND_CONV, OpNode
from .ndarray import NdArray, nda_from_np
from .variants import STATIC, KernelPlan, TuneParams, Variant, conv_shape


def seed_for(signature: str) -> int:
    """Process-independent 64-bit seed: first 8 bytes (LE) of sha256 (oracle.py:48-50)."""
    return int.from_bytes(hashlib.sha256(signature.encode()).digest()[:8], "little")


def noise(names, sizes, seed: int, low: float = 0.1, high: float = 1.0) -> NdArray:
    """Uniform fp32 synthetic data; [0.1, 1) is the reference recipe (oracle.py:53-60)."""
    n = int(np.prod(sizes, dtype=np.int64))
    vals = np.random.default_rng(seed).uniform(low, high, size=n).astype(np.float32)
    return nda_from_np(names, vals.reshape(tuple(sizes)))


def node_test_inputs(node: OpNode, edges, seed, low: float = 0.1, high: float = 1.0) -> dict:
    """Seeded noise for every input edge of a node, seed ``f"{seed}:{edge}"`` (runner.py:39-45)."""
    return {e: noise(edges[e].names, edges[e].sizes, seed_for(f"{seed}:{e}"), low, high) for e in node.inputs}


def conv_reduction_terms(node: OpNode, edges) -> int:
    """ic*k*k, the reduction length that picks the tolerance (runner.py:66-70)."""
    if node.kind != KIND_CONV:
        return 1
    return edges[node.inputs[0]].size_of("chan") * node.params.ksz ** 2


def _torch():
    import torch

    if not torch.cuda.is_available():
        from .errors import DeviceError

        raise DeviceError("no CUDA device: the B200 conv path has no CPU fallback")
    return torch


class ConvOp:
    """One conv bound to device operands and a kernel plan; ``launch()`` = one kernel.

    Filters are constant per op: at construction the tcgen05 variants pack them
    once into the workspace (b2c_conv_prepare — the cached filter transform of
    SURVEY.md §8(b); the reference's ConvTiled asks for re-laid-out filters via
    required_formats, variants.py:416-424).  ``prepare()`` re-packs after the
    filter tensor changes."""

    def __init__(self, plan: KernelPlan, x, w, bias, y=None, device=None):
        torch = _torch()
        self.plan = plan
        d = plan.desc
        dev = device or x.device
        for t, shape in ((x, (d.n, d.c, d.h, d.w)), (w, (d.k, d.c, d.r, d.r)), (bias, (d.k,))):
            if tuple(t.shape) != shape or t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
                raise CuclgenError(f"operand {tuple(t.shape)} {t.dtype} does not match {shape} fp32 contiguous CUDA")
        self.x, self.w, self.bias = x, w, bias
        self.y = y if y is not None else torch.empty((d.n, d.k, d.oh, d.ow), dtype=torch.float32, device=dev)
        self.ws = backend.alloc_workspace(d, plan.tune, device=dev)
        self.tune = backend.Tune.from_buffer_copy(plan.tune)
        self.prepare()

    def prepare(self, stream=None):
        """Pack the filters (tcgen05 variants) and mark the plan prepared."""
        self.tune.prepared = 0
        backend.prepare(self.plan.desc, self.tune, self.w, self.ws, stream)
        self.tune.prepared = 1

    @property
    def flops(self) -> int:
        return backend.conv_flops(self.plan.desc)

    @property
    def bytes(self) -> int:
        return backend.conv_bytes(self.plan.desc)

    def launch(self, stream=None):
        backend.fwd(self.plan.desc, self.tune, self.x, self.w, self.bias, self.y, self.ws, stream)

    def time_ms(self, warmup=3, reps=10, l2_flush=True) -> float:
        return backend.time_ms(self.plan.desc, self.tune, self.x, self.w, self.bias, self.y, self.ws,
                               warmup, reps, l2_flush)

    def prepare_ms(self) -> float:
        """Device time of one filter pack (0 for variants that need none)."""
        torch = _torch()
        if self.ws is None:
            return 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        self.prepare()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1)


def to_device(nda: NdArray, device="cuda"):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(nda.to_np())).to(device)


def execute_node(node: OpNode, edges, inputs: dict, variant: Variant, params: TuneParams | None = None,
                 mode: str = STATIC, engine=None, thread_order=None, inst: KernelPlan | None = None, src=None):
    """Run one node's kernel on canonical inputs; returns (canonical output NdArray,
    CostReport) like runner.execute_node (runner.py:73-106).  ``engine`` /
    ``thread_order`` / ``src`` belong to the reference's simulator and are
    accepted for signature compatibility only."""
    torch = _torch()
    if params is None:
        params = variant.default_params(node, edges)
    plan = inst if inst is not None else variant.generate(node, edges, params, mode)
    x, w, b = (to_device(inputs[e]) for e in node.inputs)
    op = ConvOp(plan, x, w, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    op.launch()
    e1.record()
    e1.synchronize()
    out_spec = edges[node.outputs[0]]
    got = op.y.cpu().numpy().reshape(out_spec.sizes)
    return nda_from_np(out_spec.names, got), CostReport(wall_ns=int(e0.elapsed_time(e1) * 1e6))


@dataclass
class HostRun:
    """Pinned host operands + device scratch for the end-to-end call
    (b2c_conv_fwd_host: H2D inputs, kernel, D2H output on one stream)."""

    plan: KernelPlan
    hx: object
    hw: object
    hb: object
    hy: object
    scratch: object

    @staticmethod
    def create(plan: KernelPlan, x_np, w_np, b_np, device="cuda") -> "HostRun":
        torch = _torch()
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).pin_memory()  # noqa: E731
        d = plan.desc
        hy = torch.empty((d.n, d.k, d.oh, d.ow), dtype=torch.float32).pin_memory()
        nbytes = backend.lib().b2c_conv_host_scratch(backend.ctypes.byref(d), backend.ctypes.byref(plan.tune))
        scratch = torch.zeros(int(nbytes), dtype=torch.uint8, device=device)
        return HostRun(plan, pin(x_np), pin(w_np), pin(b_np), hy, scratch)

    @property
    def h2d_bytes(self) -> int:
        return 4 * (self.hx.numel() + self.hw.numel() + self.hb.numel())

    @property
    def d2h_bytes(self) -> int:
        return 4 * self.hy.numel()

    def run(self, stream=None):
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        L = backend.lib()
        rc = L.b2c_conv_fwd_host(backend.ctypes.byref(self.plan.desc), backend.ctypes.byref(self.plan.tune),
                                 self.hx.data_ptr(), self.hw.data_ptr(), self.hb.data_ptr(), self.hy.data_ptr(),
                                 self.scratch.data_ptr(), self.scratch.numel(), st)
        backend.check(rc, "b2c_conv_fwd_host")


def shape_of(node: OpNode, edges):
    return conv_shape(node, edges)


# ============================================================================ whole-network forward
# plan_graph / run_graph (cuclgen/runner.py:118-249) on
# the B200.  Every node is one launch of a libb2conv kernel on one stream, so a
# whole forward pass can be captured in a CUDA graph (GraphExec.launch).


@dataclass
class ExecPlan:
    """Variant choices, kernel plans and the conversion-spliced graph
    (runner.py:118-152)."""

    graph: object
    pre_graph: object
    order: list
    alloc: object
    insts: dict
    choices: dict
    canonical_inputs: dict
    canonical_output: dict


@dataclass
class NodeRun:
    name: str
    variant: str
    params: object
    report: CostReport
    cost: float


@dataclass
class RunResult:
    checksums: dict
    node_runs: list = None
    oracle_checks: dict = None
    sink_buffers: dict = None

    def __post_init__(self):
        self.node_runs = [] if self.node_runs is None else self.node_runs
        self.oracle_checks = {} if self.oracle_checks is None else self.oracle_checks
        self.sink_buffers = {} if self.sink_buffers is None else self.sink_buffers


def plan_graph(g, db=None, fuse: bool = True, prec: int | None = None) -> ExecPlan:
    """fuse_activations, per-node select_variant + generate, insert_conversions
    for the variants' required formats (Xpose nodes for the conversions), then
    schedule and allocate (runner.py:155-193).  ``prec`` pins the conv nodes'
    precision mode (None: whatever the DB records say)."""
    from . import graphopt
    from .frontend import KIND_CONV, KIND_CONVERT, KIND_INPUT
    from .variants import DEFAULT_TUNE, VARIANTS, select_variant

    if fuse:
        g = graphopt.fuse_activations(g)
    choices, fmts, insts, cin, cout = {}, {}, {}, {}, {}
    for n in g.nodes:
        if n.kind == KIND_INPUT:
            continue
        v, p = select_variant(n, g.edges, db, prec=prec if n.kind == KIND_CONV else None)
        choices[n.name] = (v, p)
        fmts[n.name] = v.required_formats(n, g.edges, p)
        insts[n.name] = v.generate(n, g.edges, p, STATIC)
        cin[n.name], cout[n.name] = n.inputs, n.outputs[0]
    g2 = graphopt.insert_conversions(g, fmts)
    for n in g2.nodes:
        if n.kind == KIND_CONVERT and n.name not in insts:
            xp = VARIANTS["xpose"]
            choices[n.name] = (xp, DEFAULT_TUNE)
            insts[n.name] = xp.generate(n, g2.edges, DEFAULT_TUNE, STATIC)
    order = [name for name in graphopt.schedule(g2) if g2.node(name).kind != KIND_INPUT]
    return ExecPlan(g2, g, order, graphopt.alloc_plan(g2), insts, {k: (v.name, p) for k, (v, p) in choices.items()},
                    cin, cout)


def checksum_bytes(buf: bytes) -> str:
    """First 16 hex digits of sha256 over the fp32 buffer (runner.py:196-197)."""
    return hashlib.sha256(buf).hexdigest()[:16]


class GraphExec:
    """A planned graph bound to device memory: one dense fp32 buffer per edge
    (alloc_plan), sources filled with the seeded reference noise
    (runner.py:213-216), conv filters packed once.  ``launch()`` issues every
    node in schedule order on one stream — capturable in a CUDA graph."""

    def __init__(self, plan: ExecPlan, seed=0, device="cuda", low: float = 0.1, high: float = 1.0):
        torch = _torch()
        from .frontend import KIND_CONV

        self.plan, g = plan, plan.graph
        self.buffers = {}
        for e, spec in g.edges.items():
            self.buffers[e] = torch.empty(spec.sizes, dtype=torch.float32, device=device)
        for e in g.sources:
            spec = g.edges[e]
            self.buffers[e].copy_(torch.from_numpy(noise(spec.names, spec.sizes, seed_for(f"{seed}:{e}"), low, high).to_np()))
        self.ops = {}
        for name in plan.order:
            node = g.node(name)
            if node.kind == KIND_CONV:
                x, w, b = (self.buffers[e] for e in node.inputs)
                self.ops[name] = ConvOp(plan.insts[name], x, w, b, y=self.buffers[node.outputs[0]])
        torch.cuda.synchronize()

    def launch_node(self, name: str, stream=None):
        node = self.plan.graph.node(name)
        if name in self.ops:
            self.ops[name].launch(stream)
            return
        inst = self.plan.insts[name]
        x, y = self.buffers[node.inputs[0]], self.buffers[node.outputs[0]]
        if inst.variant == "pool_max":
            backend.pool_max_fwd(inst.desc, x, y, stream)
        elif inst.variant == "activation":
            backend.relu_fwd(x, y, stream)
        elif inst.variant == "xpose":
            backend.xpose(inst.desc, x, y, stream)
        else:
            raise CuclgenError(f"node '{name}': no launcher for variant {inst.variant}")

    def launch(self, stream=None):
        for name in self.plan.order:
            self.launch_node(name, stream)

    def nda(self, edge: str) -> NdArray:
        spec = self.plan.graph.edges[edge]
        return nda_from_np(spec.names, self.buffers[edge].cpu().numpy())

    @property
    def flops(self) -> int:
        return sum(op.flops for op in self.ops.values())


def run_graph(g, seed=0, db=None, check=None, fuse: bool = True, engine=None, keep_sinks: bool = False,
              prec: int | None = None) -> RunResult:
    """Execute a whole graph on the B200 (runner.py:200-249): plan, allocate,
    fill sources with seeded noise, launch every node in schedule order (each
    timed with CUDA events into its CostReport), then checksum the sinks.

    ``check``: the reference compares each node with its CPU oracle; the product
    ships no CPU path, so the caller supplies the checker —
    ``check(node, edges, inputs: dict[edge, NdArray], got: NdArray) -> result``
    — and its results land in ``RunResult.oracle_checks``.  Each node is
    checked against its canonical (pre-conversion) operand edges.  ``engine``
    belongs to the reference's simulator and is accepted for signature
    compatibility only."""
    torch = _torch()
    from dataclasses import replace as dc_replace

    plan = plan_graph(g, db=db, fuse=fuse, prec=prec)
    ex = GraphExec(plan, seed)
    res = RunResult(checksums={})
    for name in plan.order:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ex.launch_node(name)
        e1.record()
        e1.synchronize()
        ns = int(e0.elapsed_time(e1) * 1e6)
        vname, params = plan.choices[name]
        res.node_runs.append(NodeRun(name, vname, params, CostReport(wall_ns=ns), float(ns)))
    if check is not None:
        g2 = plan.graph
        for name in plan.order:
            node = g2.node(name)
            if name in plan.canonical_inputs:
                node = dc_replace(node, inputs=plan.canonical_inputs[name], outputs=(plan.canonical_output[name],))
            inputs = {e: ex.nda(e) for e in node.inputs}
            res.oracle_checks[name] = check(node, g2.edges, inputs, ex.nda(node.outputs[0]))
    for e in plan.graph.sinks:
        arr = ex.buffers[e].cpu().numpy()
        res.checksums[e] = checksum_bytes(arr.tobytes())
        if keep_sinks:
            res.sink_buffers[e] = nda_from_np(plan.graph.edges[e].names, arr)
    return res
