"""Per-shape autotuning timed on the B200, with the reference's tuning-DB contract.

Mirrors cuclgen/tuner.py: ``op_signature`` (tuner.py:66-89), ``TuneSpace`` /
``default_space`` (:190-212), ``TuneRecord`` / ``TuneDB`` / ``save_db`` /
``load_db`` with the ``boda-tunedb v1`` TSV format and atomic save
(:219-294), ``sweep`` (:331-378) and ``tune_all`` (:381-398), including the
argmin rule (cost, then enumeration index — most specialized variant first)
and ``AllCandidatesFailed``.

What changes:
* candidates are validated at the TRUE shape on the device, not on a
  downscaled twin: each candidate's output is compared with the exact-order
  ``conv_simple`` kernel's output at the reference tolerance
  (oracle.tolerance_for, oracle.py:31-38) — a device-side check, the CPU
  oracle stays test-only;
* the objective is ``wall``: median CUDA-event time of the kernel with the
  L2 flushed before every rep; the simulator's counter ``model`` objective
  has no B200 meaning and is rejected.
"""

from __future__ import annotations

import logging
import os
import tempfile
from dataclasses import dataclass, field

from .backend import CostReport
from .errors import CuclgenError, Inapplicable
from .frontend import KIND_ACT, KIND_CONV, KIND_CONVERT, KIND_POOL, ConvParams, OpNode, window_out
from .variants import VARIANTS, TuneParams, variants_for_kind

log = logging.getLogger(__name__)

DB_HEADER = "boda-tunedb v1"
MODEL = "model"
WALL = "wall"
LONG_REDUCTION_TERMS = 4096


class AllCandidatesFailed(CuclgenError):
    pass


class IoError(CuclgenError):
    pass


class FormatVersionMismatch(CuclgenError):
    pass


def op_signature(node: OpNode, edges) -> str:
    """Canonical per-op key (tuner.py:66-89): ``conv:k{k}:s{s}:p{p}:oc{oc}:in{b}x{ic}x{h}x{w}[:relu]``,
    ``pool_max:k..:s..:p..:in{b}x{c}x{h}x{w}``, ``relu:in{dims}``, ``xpose:{src}-to-{dst}``."""
    if node.kind == KIND_CONV:
        p = node.params
        b, ic, h, w = edges[node.inputs[0]].sizes
        sig = f"conv:k{p.ksz}:s{p.stride}:p{p.pad}:oc{p.out_chans}:in{b}x{ic}x{h}x{w}"
        return sig + (f":{node.fused_activation}" if node.fused_activation else "")
    if node.kind == KIND_POOL:
        p = node.params
        b, c, h, w = edges[node.inputs[0]].sizes
        return f"pool_max:k{p.ksz}:s{p.stride}:p{p.pad}:in{b}x{c}x{h}x{w}"
    if node.kind == KIND_ACT:
        return "relu:in" + "x".join(str(s) for s in edges[node.inputs[0]].sizes)
    if node.kind == KIND_CONVERT:
        fmt = lambda s: "_".join(f"{n}{v}" for n, v in zip(s.names, s.sizes))  # noqa: E731
        return f"xpose:{fmt(edges[node.inputs[0]])}-to-{fmt(edges[node.outputs[0]])}"
    raise CuclgenError(f"no signature for kind {node.kind}")


def conv_flops(p: ConvParams, b: int, ic: int, h: int, w: int) -> int:
    oy, ox = window_out(h, p.ksz, p.stride, p.pad), window_out(w, p.ksz, p.stride, p.pad)
    return 2 * p.ksz * p.ksz * ic * p.out_chans * oy * ox * b


@dataclass(frozen=True)
class ToleranceSpec:
    rel_tol: float = 1e-5
    abs_floor: float = 1e-6


BF16_REL_TOL = 4e-3  # bf16 operands, fp32 accumulate
FP8_REL_TOL = 0.13  # e4m3 operands: <= 2*2^-4 + 2^-8 relative per product (rigorous on U[0.1, 1) data), fp32 accumulate


def tolerance_for(reduction_terms: int, prec: int = 0) -> ToleranceSpec:
    """rel 1e-5 up to 4096 reduction terms, 1e-3 beyond (oracle.py:31-38); the
    separately stated bf16-mode tolerance is rel 4e-3."""
    if prec == 1:
        return ToleranceSpec(rel_tol=BF16_REL_TOL)
    if prec == 2:
        return ToleranceSpec(rel_tol=FP8_REL_TOL)
    return ToleranceSpec(rel_tol=1e-3) if reduction_terms > LONG_REDUCTION_TERMS else ToleranceSpec()


def device_compare(got, want, tol: ToleranceSpec):
    """(ok, max_rel_err) of |a-b| <= max(floor, rel*max(|a|,|b|)) on device tensors
    (the compare rule of oracle.py:124-137, evaluated by torch on the GPU)."""
    import torch

    a, b = got.double(), want.double()
    diff = (a - b).abs()
    mag = torch.maximum(a.abs(), b.abs())
    ok = bool((diff <= torch.clamp(tol.rel_tol * mag, min=tol.abs_floor)).all().item())
    rel = torch.where(mag > 0, diff / mag, torch.zeros_like(diff))
    return ok and bool(torch.isfinite(a).all().item()), float(rel.max().item()) if rel.numel() else 0.0


@dataclass(frozen=True)
class TuneSpace:
    """Optional per-variant candidate override: {variant name: (TuneParams, ...)}.
    Variants absent from the mapping use their own B200 space."""

    per_variant: dict = field(default_factory=dict)


def default_space() -> TuneSpace:
    return TuneSpace()


@dataclass
class TuneRecord:
    op_signature: str
    variant: str
    params: TuneParams
    cost: float
    counters: CostReport
    objective: str = WALL
    scoring: str = "device-wall"
    timestamp: float = 0.0
    max_rel_err: float = 0.0

    def line(self) -> str:
        c = int(self.cost) if float(self.cost).is_integer() else self.cost
        return f"{self.op_signature}\t{self.variant}\t{self.params.to_string()}\t{c}\t{self.objective}"


@dataclass
class TuneDB:
    records: dict = field(default_factory=dict)

    def add(self, rec: TuneRecord):
        self.records[rec.op_signature] = rec

    def persisted(self) -> tuple:
        return tuple(sorted(r.line() for r in self.records.values()))

    def __eq__(self, other):
        return isinstance(other, TuneDB) and self.persisted() == other.persisted()


def save_db(db: TuneDB, path):
    """Atomic: write a temp file beside the target, then rename (tuner.py:249-260)."""
    path = os.fspath(path)
    body = DB_HEADER + "\n" + "".join(f"{ln}\n" for ln in db.persisted())
    try:
        fd, tmp = tempfile.mkstemp(prefix=".tunedb-", dir=os.path.dirname(path) or ".")
        with os.fdopen(fd, "w") as fh:
            fh.write(body)
        os.replace(tmp, path)
    except OSError as e:
        raise IoError(f"cannot write {path}: {e}") from None


def load_db(path) -> TuneDB:
    path = os.fspath(path)
    try:
        with open(path, encoding="utf-8") as fh:
            lines = fh.read().splitlines()
    except OSError as e:
        raise IoError(f"cannot read {path}: {e}") from None
    if not lines or lines[0] != DB_HEADER:
        raise FormatVersionMismatch(f"{path}: expected header {DB_HEADER!r}")
    db = TuneDB()
    for ln in filter(str.strip, lines[1:]):
        parts = ln.split("\t")
        if len(parts) != 5 or parts[1] not in VARIANTS or parts[4] not in (MODEL, WALL):
            raise FormatVersionMismatch(f"{path}: malformed record {ln!r}")
        sig, variant, params_s, cost_s, objective = parts
        try:
            cost = float(cost_s) if any(ch in cost_s for ch in ".eE") else int(cost_s)
        except ValueError:
            raise FormatVersionMismatch(f"{path}: bad cost in {ln!r}") from None
        try:
            params = TuneParams.from_string(params_s)
        except CuclgenError:
            raise FormatVersionMismatch(f"{path}: bad params in {ln!r}") from None
        db.add(TuneRecord(sig, variant, params, cost, CostReport(), objective=objective, scoring="loaded"))
    return db


def candidates(node: OpNode, edges, space: TuneSpace | None = None, prec: int = 0) -> list:
    """All applicable (variant, params), most specialized variant first (tuner.py:301-308).
    ``prec`` 1 re-targets every candidate to the bf16 mode (TuneParams.prec) and keeps
    the applicable ones."""
    from .variants import with_prec

    space = space or default_space()
    out = []
    for v in variants_for_kind(node.kind):
        plist = space.per_variant.get(v.name)
        if plist is None:
            plist = v.space(node, edges, prec)  # the variant's own space, built and filtered in mode `prec`
        else:
            plist = with_prec(list(plist), prec) if prec else list(plist)
        out.extend((v, p) for p in v.tune_candidates(node, edges, plist))
    return out


def sweep(node: OpNode, edges, space: TuneSpace | None = None, objective: str = WALL, reps: int = 5,
          warmup: int = 2, l2_flush: bool = True, seed: str = "validate", jobs: int = 1, prec: int = 0,
          record_all: list | None = None) -> TuneRecord:
    """Time every applicable candidate on the device and return the fastest one
    that matches the exact-order conv_simple output within tolerance.  Ties
    break by enumeration order (specialized variants first), tuner.py:367-373."""
    if objective != WALL:
        raise CuclgenError("objective 'model' is the simulator's counter model; the B200 tuner times on device ('wall')")
    if node.kind != KIND_CONV:
        raise AllCandidatesFailed(f"no variant applies to '{node.name}'")
    cands = candidates(node, edges, space, prec)
    if not cands:
        raise AllCandidatesFailed(f"no variant applies to '{node.name}'")
    import torch

    from .runner import ConvOp, node_test_inputs, to_device

    inputs = node_test_inputs(node, edges, seed)
    x, w, b = (to_device(inputs[e]) for e in node.inputs)
    ref_plan = VARIANTS["conv_simple"].generate(node, edges, TuneParams())
    ref = ConvOp(ref_plan, x, w, b)
    ref.launch()
    torch.cuda.synchronize()
    tol = tolerance_for(edges[node.inputs[0]].size_of("chan") * node.params.ksz ** 2, prec)
    sig = op_signature(node, edges)
    best, best_key, failures = None, None, []
    for idx, (v, params) in enumerate(cands):
        try:
            op = ConvOp(v.generate(node, edges, params), x, w, b)
            op.y.fill_(float("nan"))
            op.launch()
            torch.cuda.synchronize()
            ok, err = device_compare(op.y, ref.y, tol)
            if not ok:
                failures.append(f"{v.name}[{params.to_string()}]: device mismatch (rel err {err:.3g})")
                continue
            ms = op.time_ms(warmup=warmup, reps=reps, l2_flush=l2_flush)
        except (Inapplicable, CuclgenError) as e:
            failures.append(f"{v.name}[{params.to_string()}]: {e}")
            continue
        rec = TuneRecord(sig, v.name, params, round(ms * 1e6, 1), CostReport(wall_ns=int(ms * 1e6)), max_rel_err=err)
        if record_all is not None:  # every valid candidate: (variant, params, ns, CTAs of the main kernel)
            from . import backend

            ctas = int(backend.lib().b2c_conv_grid(backend.ctypes.byref(op.plan.desc), backend.ctypes.byref(op.plan.tune)))
            record_all.append((sig, v.name, params.to_string(), rec.cost, ctas))
        key = (rec.cost, idx)
        if best is None or key < best_key:
            best, best_key = rec, key
    if best is None:
        raise AllCandidatesFailed(f"every candidate for '{node.name}' failed:\n  " + "\n  ".join(failures))
    if failures:
        log.debug("sweep '%s': %d candidates rejected", node.name, len(failures))
    return best


def tune_all(nodes_and_edges, space: TuneSpace | None = None, **kw) -> TuneDB:
    """One sweep per distinct signature (tuner.py:381-398); takes (node, edges) pairs."""
    db = TuneDB()
    for node, edges in nodes_and_edges:
        if node.kind != KIND_CONV:
            continue
        sig = op_signature(node, edges)
        if sig not in db.records:
            db.add(sweep(node, edges, space, **kw))
    return db


def shipped_db_path(prec: str = "fp32") -> str:
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", f"tunedb_b200_{prec}.tsv")
