"""Conv variants and their tuning parameters — the reference's variant API on B200.

Mirrors cuclgen/variants.py: ``TuneParams`` (variants.py:39-91) with the same
string form, the ``Variant`` protocol (``applies`` / ``required_formats`` /
``generate`` / ``tune_candidates``, variants.py:201-220), the ``VARIANTS``
registry (:830-832), ``variants_for_kind`` (:835-837) and ``select_variant``
(:840-856: a TuneDB record wins, else the most specialized applicable variant).

What changes is what ``generate`` produces.  The reference emits CUCL kernel
text for its SIMT interpreter; here a variant resolves to one of the
hand-written sm_100a kernels in libb2conv.so and ``generate`` returns the
launch plan (C descriptor + tune struct) the C ABI executes:

    conv_simple  one thread per output, exact fmaf order     (variants.py:223-276)
    conv_tiled   FFMA register/thread-blocked implicit GEMM  (variants.py:376-685)
    conv_umma    tcgen05/TMEM 3xTF32 implicit GEMM, k x k     (new)
    conv_1x1     tcgen05 GEMM for k=1, pad=0                 (variants.py:279-325)
    conv_fc      tcgen05 weight-streaming GEMM, k = h = w     (variants.py:328-373)

Every kernel reads canonical NCHW / OIHW and writes NCHW, so
``required_formats`` is canonical for all of them (no conversion passes,
unlike ConvTiled's padded NHWC output, variants.py:416-424).

The non-conv kinds of a whole-network run are variants too,
each bound to a libb2conv kernel:

    pool_max     window max, -inf padding                    (variants.py:688-741)
    activation   ReLU                                        (variants.py:744-775)
    xpose        layout conversion: permute / pad / crop     (variants.py:778-827)
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import backend
from .errors import CuclgenError, Inapplicable
from .frontend import KIND_ACT, KIND_CONV, KIND_CONVERT, KIND_POOL, OpNode
from .graphopt import VariantFormats

STATIC = "static"
DYNAMIC = "dynamic"

UMMA_BN = (16, 32, 64, 96, 128, 192)  # 16: the swapped fc tile (batch <= 16)
NUM_SMS = 148


@dataclass(frozen=True)
class TuneParams:
    """The reference knobs (MNt register block, MNb thread block, Kb reduction
    chunk, vw vector width, lf/li staging flags) plus the tcgen05 knobs:
    bn (MMA N tile), split_k, swap_ab (M = out_chans instead of pixels)."""

    mnt: tuple = (4, 4)
    mnb: tuple = (16, 16)
    kb: int = 4
    vw: int = 4
    use_local_filts: bool = True
    use_local_in: bool = True
    bn: int = 128
    split_k: int = 1
    swap_ab: bool = False
    drain: int = 0  # K blocks per TMEM chunk before the fp32 register drain (0 = library default)
    tma: int = 0  # tcgen05: 1 = TMA-fed kernel (im2col on an NHWC copy / 2-D tiles), 2 = 2-D tiles for 1x1; 0 = warp gathers
    occ: int = 1  # TMA kernel: CTAs per SM (2 needs bn <= 64)
    cl: int = 1  # TMA kernel: 2 = CTA pairs sharing (multicasting) the filter stages
    prec: int = 0  # 0 fp32-exact (default), 1 bf16 operands / fp32 accumulate (TMA tcgen05 kernel only)

    def __post_init__(self):
        if min(self.mnt) < 1 or min(self.mnb) < 1 or self.kb < 1:
            raise CuclgenError(f"bad tune params {self}")
        if self.threads > 1024:
            raise CuclgenError(f"workgroup of {self.threads} threads exceeds 1024")
        if self.vw not in (1, 2, 4, 8):
            raise CuclgenError(f"vector width must be one of 1,2,4,8, got {self.vw}")
        if self.mnt[1] % self.vw:
            raise CuclgenError(f"vector width {self.vw} must divide register block {self.mnt[1]}")
        if self.bn < 1 or self.split_k < 0 or self.drain < 0:  # split_k 0 = stream-K (TMA kernel)
            raise CuclgenError(f"bad tcgen05 tile params {self}")

    @property
    def threads(self) -> int:
        return self.mnb[0] * self.mnb[1]

    def to_string(self) -> str:
        return (f"MNt={self.mnt[0]}:{self.mnt[1]},MNb={self.mnb[0]}:{self.mnb[1]},Kb={self.kb},vw={self.vw},"
                f"lf={int(self.use_local_filts)},li={int(self.use_local_in)},"
                f"BN={self.bn},sk={self.split_k},sw={int(self.swap_ab)},dr={self.drain}"
                + (f",tm={int(self.tma)}" if self.tma else "") + (f",oc={self.occ}" if self.occ != 1 else "") + (f",cl={self.cl}" if self.cl != 1 else "")
                + (f",pr={self.prec}" if self.prec else ""))

    @staticmethod
    def from_string(text: str) -> "TuneParams":
        """Parses the reference form (variants.py:73-91); the tcgen05 keys are optional."""
        kv = dict(part.partition("=")[::2] for part in text.split(","))
        try:
            return TuneParams(
                mnt=tuple(int(v) for v in kv["MNt"].split(":")),
                mnb=tuple(int(v) for v in kv["MNb"].split(":")),
                kb=int(kv["Kb"]),
                vw=int(kv["vw"]),
                use_local_filts=kv.get("lf", "1") == "1",
                use_local_in=kv.get("li", "1") == "1",
                bn=int(kv.get("BN", "128")),
                split_k=int(kv.get("sk", "1")),
                swap_ab=kv.get("sw", "0") == "1",
                drain=int(kv.get("dr", "0")),
                tma=int(kv.get("tm", "0")),
                occ=int(kv.get("oc", "1")),
                cl=int(kv.get("cl", "1")),
                prec=int(kv.get("pr", "0")),
            )
        except (KeyError, ValueError) as e:
            raise CuclgenError(f"bad tune-params string {text!r}: {e}") from None


DEFAULT_TUNE = TuneParams()


@dataclass(frozen=True)
class ConvShape:
    b: int
    ic: int
    h: int
    w: int
    oc: int
    oy: int
    ox: int
    ksz: int
    stride: int
    pad: int

    @property
    def m(self) -> int:
        return self.b * self.oy * self.ox

    @property
    def k(self) -> int:
        return self.ic * self.ksz * self.ksz


def conv_shape(node: OpNode, edges) -> ConvShape:
    ind, outd = edges[node.inputs[0]], edges[node.outputs[0]]
    if ind is None or outd is None:
        raise CuclgenError(f"node '{node.name}': shapes not inferred")
    p = node.params
    b, ic, h, w = (ind.size_of(d) for d in ("img", "chan", "y", "x"))
    return ConvShape(b, ic, h, w, outd.size_of("chan"), outd.size_of("y"), outd.size_of("x"), p.ksz, p.stride, p.pad)


def conv_desc(node: OpNode, edges, prec: int = backend.PREC_FP32) -> backend.ConvDesc:
    s = conv_shape(node, edges)
    act = node.fused_activation
    if act not in (None, "relu"):
        raise Inapplicable(f"no fused form for activation '{act}'")
    return backend.make_desc(s.b, s.ic, s.h, s.w, s.oc, s.ksz, s.stride, s.pad, s.oy, s.ox, act == "relu", prec)


@dataclass(frozen=True)
class KernelPlan:
    """What ``generate`` returns: the C launch description of one op."""

    variant: str
    desc: backend.ConvDesc
    tune: backend.Tune
    params: TuneParams

    @property
    def name(self) -> str:
        d = self.desc
        return f"{self.variant}_b{d.n}_ic{d.c}_y{d.h}_x{d.w}_oc{d.k}_k{d.r}_s{d.stride}_p{d.pad}"


class Variant:
    name: str
    rank: int
    kind: str = KIND_CONV
    vid: int

    def tune_struct(self, params: TuneParams) -> backend.Tune:
        return backend.Tune(self.vid, params.mnt[0], params.mnt[1], params.mnb[0], params.mnb[1], params.kb,
                            params.vw, params.bn, params.occ if params.tma else 0, params.split_k,
                            int(params.swap_ab), params.drain, 0, int(params.tma), params.cl)

    def applies(self, node: OpNode, edges, params: TuneParams) -> str | None:
        """None when applicable, else the reason (variants.py:206-210).  The C
        library's b2c_conv_applies is the single source of truth."""
        if node.kind != self.kind:
            return f"kind {node.kind} != {self.kind}"
        if node.fused_activation not in (None, "relu"):
            return f"no fused form for activation '{node.fused_activation}'"
        return backend.applies(conv_desc(node, edges, params.prec), self.tune_struct(params))

    def required_formats(self, node: OpNode, edges, params: TuneParams) -> VariantFormats:
        return VariantFormats()

    def default_params(self, node: OpNode, edges) -> TuneParams:
        return DEFAULT_TUNE

    def space(self, node: OpNode, edges, prec: int = 0) -> list:
        """This variant's own candidate list for the on-device sweep, in precision mode ``prec``
        (candidates are filtered by applicability in that mode)."""
        p = self.default_params(node, edges)
        if prec:
            from dataclasses import replace

            p = replace(p, prec=prec)
        return [p] if self.applies(node, edges, p) is None else []

    def tune_candidates(self, node: OpNode, edges, candidates):
        return [p for p in candidates if self.applies(node, edges, p) is None]

    def generate(self, node: OpNode, edges, params: TuneParams, mode: str = STATIC) -> KernelPlan:
        reason = self.applies(node, edges, params)
        if reason:
            raise Inapplicable(f"{self.name} on '{node.name}': {reason}")
        return KernelPlan(self.name, conv_desc(node, edges, params.prec), self.tune_struct(params), params)


class ConvSimple(Variant):
    name, rank, vid = "conv_simple", 0, backend.VAR_SIMPLE


class ConvTiled(Variant):
    name, rank, vid = "conv_tiled", 1, backend.VAR_TILED

    def space(self, node, edges, prec: int = 0):
        if prec:
            return []  # FFMA kernels are fp32-exact only
        out = []
        for mnt in ((4, 4), (8, 8), (8, 4), (4, 8)):
            for mnb in ((16, 16), (32, 8), (8, 32), (16, 8)):
                for kb in (8, 16):
                    out.append(TuneParams(mnt=mnt, mnb=mnb, kb=kb, vw=4))
        return [p for p in out if self.applies(node, edges, p) is None]


def _ceil(a: int, b: int) -> int:
    return -(-a // b)


class _UmmaFamily(Variant):
    """tcgen05 3xTF32 implicit GEMM; ``kmode`` is fixed per registered name."""

    def default_params(self, node, edges):
        s = conv_shape(node, edges)
        kblocks = _ceil(s.k, 32)

        def plan(swap, bn):
            rows_m, rows_n = (s.oc, s.m) if swap else (s.m, s.oc)
            tiles = _ceil(rows_m, 128) * _ceil(rows_n, bn)
            waste = _ceil(rows_m, 128) * 128 * _ceil(rows_n, bn) * bn
            return tiles, waste

        best = None
        for swap in (False, True):
            for bn in UMMA_BN:
                if bn < 32:  # (16: a tuner-only fc tile)
                    continue
                tiles, waste = plan(swap, bn)
                key = (waste, -bn)
                if best is None or key < best[0]:
                    best = (key, swap, bn, tiles)
        _, swap, bn, tiles = best
        split = 1
        while tiles * split * 2 <= NUM_SMS and kblocks // (split * 2) >= 4:
            split *= 2
        p = TuneParams(bn=bn, split_k=split, swap_ab=swap, tma=1)
        if self.applies(node, edges, p) is None:
            return p
        return TuneParams(bn=bn, split_k=split, swap_ab=swap)

    def space(self, node, edges, prec: int = 0):
        from dataclasses import replace

        s = conv_shape(node, edges)
        kblocks = _ceil(s.k, 32)
        out = []
        for swap in (False, True):
            n_rows = s.m if swap else s.oc
            for bn in UMMA_BN:
                if bn > 2 * max(32, n_rows):
                    continue
                for split in (1, 2, 4, 8, 16, 32, 0):  # 0 = stream-K (TMA kernel)
                    if split > 1 and kblocks // split < 2:
                        continue
                    for tma in ((1, 2, 3, 4, 5, 6) if split == 0 else (1, 2, 3, 4, 5, 6, 0)):  # 5: bf16 mode only; 6: first layers
                        out.append(TuneParams(bn=bn, split_k=split, swap_ab=swap, tma=tma))
                        if tma and split and bn <= 64:  # two CTAs per SM
                            out.append(TuneParams(bn=bn, split_k=split, swap_ab=swap, tma=tma, occ=2))
                        if tma in (1, 2) and split and bn >= 64 and not swap:  # CTA pairs multicasting filters
                            out.append(TuneParams(bn=bn, split_k=split, swap_ab=swap, tma=tma, cl=2))
                        if (tma in (1, 3, 4, 6) and bn in (64, 96, 128, 192) or tma == 5 and bn in (128, 192)) and not swap:  # 2-SM UMMA pairs (M = 256)
                            out.append(TuneParams(bn=bn, split_k=split, swap_ab=swap, tma=tma, cl=3))
                        if 2 <= split <= 8 and tma in (1, 3, 4) and (bn in (32, 64) and not swap or bn == 32 and swap):
                            out.append(TuneParams(bn=bn, split_k=split, swap_ab=swap, tma=tma, cl=4))  # split-K cluster
        if prec:
            out = [replace(p, prec=prec) for p in out]
        return [p for p in out if self.applies(node, edges, p) is None]


def with_prec(params_list, prec: int) -> list:
    """The same candidates in another precision mode (TuneParams.prec)."""
    from dataclasses import replace

    return [replace(p, prec=prec) for p in params_list]


class ConvUmma(_UmmaFamily):
    name, rank, vid = "conv_umma", 2, backend.VAR_UMMA


class Conv1x1(_UmmaFamily):
    name, rank, vid = "conv_1x1", 3, backend.VAR_1X1


class ConvFC(_UmmaFamily):
    name, rank, vid = "conv_fc", 4, backend.VAR_FC


class ConvWino(Variant):
    """Winograd F(2x2,3x3) (the paper's gap to cuDNN on
    3x3): for 3x3, stride-1, pad <= 1 convs, 16 batched tcgen05
    3xTF32 GEMMs between the transformed input tiles V = B^T d B and the
    transformed filters U = G g G^T (built once by b2c_conv_prepare), then
    y = A^T M A + bias, ReLU.  2.25x fewer multiplies than direct conv; the
    transforms are exact-coefficient fp32 adds, so the fp32 reference tolerance
    applies unchanged.  Knobs: bn (GEMM N tile 64|128|192), split_k (0 =
    stream-K), swap_ab."""

    name, rank, vid = "conv_wino", 1, backend.VAR_WINO

    def default_params(self, node, edges):
        return TuneParams(bn=128, split_k=1, tma=1)

    def space(self, node, edges, prec: int = 0):
        if prec:
            return []  # fp32-exact only
        out = [TuneParams(bn=bn, split_k=sk, swap_ab=sw, tma=1) for sw in (False, True) for bn in (64, 128, 192)
               for sk in (1, 2, 4, 0)]
        return [p for p in out if self.applies(node, edges, p) is None]


class ConvFCStream(Variant):
    """ConvFC (variants.py:328-373) as an fp32 FFMA weight-streaming kernel for
    small batch, where the op is HBM-bound.  Kb=1 (batch <= 8): warps split K,
    x read through L1/L2, MNb0 = warps per block (2|4|8), MNt1 = rows per block
    (2|4|8).  Kb=2 (batch <= 32): x staged in shared memory per block, MNb0 =
    warps (4|8), MNt1 = rows per warp (1|2|4).  Kb=3 (batch <= 8): weights and
    x streamed by TMA bulk copies into a deep shared-memory ring (k_fc_bulk, one
    CTA per SM; MNb / MNt unused)."""

    name, rank, vid = "conv_fc_stream", 5, backend.VAR_FC_STREAM

    def default_params(self, node, edges):
        return TuneParams(mnt=(1, 4), mnb=(8, 1), kb=1, vw=1)

    def space(self, node, edges, prec: int = 0):
        if prec:
            return []  # fp32-exact only
        out = [TuneParams(mnt=(1, r), mnb=(wp, 1), kb=1, vw=1) for wp in (2, 4, 8) for r in (2, 4, 8)]
        out += [TuneParams(mnt=(1, r), mnb=(wp, 1), kb=2, vw=1) for wp in (4, 8) for r in (1, 2, 4)]
        out.append(TuneParams(mnt=(1, 1), mnb=(8, 1), kb=3, vw=1))
        return [p for p in out if self.applies(node, edges, p) is None]


@dataclass(frozen=True)
class NodePlan:
    """What ``generate`` returns for a non-conv node: the C descriptor of one
    pool / ReLU / conversion launch (``desc`` is a PoolDesc, an element count,
    or an XposeDesc)."""

    variant: str
    kind: str
    desc: object
    params: TuneParams

    @property
    def name(self) -> str:
        return f"{self.variant}_{self.kind.lower()}"


class _NodeVariant(Variant):
    """One fixed kernel per node kind; TuneParams are accepted and ignored."""

    rank = 0

    def applies(self, node, edges, params):
        if node.kind != self.kind:
            return f"kind {node.kind} != {self.kind}"
        return self._why_not(node, edges)

    def _why_not(self, node, edges):
        return None

    def generate(self, node, edges, params=None, mode: str = STATIC) -> NodePlan:
        reason = self.applies(node, edges, params)
        if reason:
            raise Inapplicable(f"{self.name} on '{node.name}': {reason}")
        return NodePlan(self.name, self.kind, self._desc(node, edges), params or DEFAULT_TUNE)


class PoolMax(_NodeVariant):
    name, kind = "pool_max", KIND_POOL

    def _desc(self, node, edges):
        i, o = edges[node.inputs[0]], edges[node.outputs[0]]
        p = node.params
        return backend.PoolDesc(*(i.size_of(d) for d in ("img", "chan", "y", "x")), p.ksz, p.stride, p.pad,
                                o.size_of("y"), o.size_of("x"))


class Activation(_NodeVariant):
    name, kind = "activation", KIND_ACT

    def _why_not(self, node, edges):
        return None if node.params.func == "relu" else f"unknown activation '{node.params.func}'"

    def _desc(self, node, edges):
        return edges[node.outputs[0]].num_elems


class Xpose(_NodeVariant):
    name, kind = "xpose", KIND_CONVERT

    def _why_not(self, node, edges):
        src, dst = edges[node.inputs[0]], edges[node.outputs[0]]
        if set(src.names) != set(dst.names):
            return f"no conversion from {src.names} to {dst.names}"
        return None

    def _desc(self, node, edges):
        src, dst = edges[node.inputs[0]], edges[node.outputs[0]]
        return backend.xpose_desc(src.names, src.sizes, [src.stride_of(n) for n in src.names], dst.names, dst.sizes)


VARIANTS: dict = {v.name: v for v in (ConvSimple(), ConvTiled(), ConvUmma(), Conv1x1(), ConvFC(), ConvFCStream(),
                                      ConvWino(), PoolMax(), Activation(), Xpose())}


def variants_for_kind(kind: str) -> list:
    """Variants for an op kind, most specialized first (variants.py:835-837)."""
    return sorted((v for v in VARIANTS.values() if v.kind == kind), key=lambda v: -v.rank)


def select_variant(node: OpNode, edges, db=None, prec: int | None = None):
    """(variant, params) for one node: the TuneDB record for its signature if
    present, else the most specialized applicable variant (variants.py:840-856).

    ``prec`` (None = whatever the record says) asks for one precision mode: a
    record of another mode is not used (op_signature carries no precision, so a
    bf16 DB handed to an fp32 run must not silently switch the arithmetic), and
    the heuristic's choice is re-targeted to that mode (first applicable
    candidate of the mode when the heuristic tile does not apply in it)."""
    from dataclasses import replace

    if db is not None:
        from .tuner import op_signature

        rec = db.records.get(op_signature(node, edges))
        if rec is not None and (prec is None or rec.params.prec == prec):
            return VARIANTS[rec.variant], rec.params
    for v in variants_for_kind(node.kind):
        params = v.default_params(node, edges)
        if prec is not None and node.kind == KIND_CONV and params.prec != prec:
            params = replace(params, prec=prec)
        if v.applies(node, edges, params) is None:
            return v, params
    if prec:  # no heuristic tile applies in this mode: the first applicable candidate of the mode
        for v in variants_for_kind(node.kind):
            for params in (v.space(node, edges, prec) if hasattr(v, "space") else []):
                if v.applies(node, edges, params) is None:
                    return v, params
    raise Inapplicable(f"no variant for node '{node.name}' of kind {node.kind}" +
                       (f" in precision mode {prec}" if prec else ""))
