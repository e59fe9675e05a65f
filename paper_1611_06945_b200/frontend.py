"""Op description: the node types of the reference front end.

The conv path mirrors ConvParams (cuclgen/frontend.py:56-65), OpNode (:93-100),
ComputeGraph (:103-159), window_out (:441-442), infer_shapes (:445-490),
flops_of (:499-514) and conv_graph (:523-532).  For whole-network runs
 it also carries PoolParams / ConvertParams
(:68-90), the layer-block network parser ``parse_net`` (:166-383: ``input:`` +
four ``input_dim:`` lines, then ``layer { ... }`` blocks of type Convolution /
Pooling (MAX) / ReLU, one bottom and one top each, unknown fields rejected)
and its inverse ``pretty_print`` (:386-434).
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field, replace

from .errors import CuclgenError
from .ndarray import DimsSpec

KIND_INPUT = "Input"
KIND_CONV = "Convolution"
KIND_POOL = "Pooling"
KIND_ACT = "Activation"
KIND_CONVERT = "Conversion"

CANONICAL_DATA_DIMS = ("img", "chan", "y", "x")
CANONICAL_FILTS_DIMS = ("out_chan", "in_chan", "y", "x")
CANONICAL_BIAS_DIMS = ("out_chan",)


class GraphError(CuclgenError):
    pass


class NetSyntaxError(CuclgenError):
    """Malformed network text (frontend.py:27-34): ``line`` and what was expected."""

    def __init__(self, line: int, expected: str, got: str = ""):
        super().__init__(f"line {line}: expected {expected}" + (f", got {got!r}" if got else ""))
        self.line, self.expected = line, expected


class UnknownLayerType(CuclgenError):
    pass


class DanglingBottom(CuclgenError):
    pass


class NonPositiveOutputDim(CuclgenError):
    def __init__(self, node: str, axis: str):
        super().__init__(f"node '{node}': non-positive output size along {axis}")
        self.node, self.axis = node, axis


@dataclass(frozen=True)
class ConvParams:
    """Square-kernel convolution: ksz, stride, pad, out_chans (frontend.py:56-65)."""

    ksz: int
    stride: int = 1
    pad: int = 0
    out_chans: int = 1

    def __post_init__(self):
        if min(self.ksz, self.stride, self.out_chans) < 1 or self.pad < 0:
            raise GraphError(f"bad conv params {self}")


@dataclass(frozen=True)
class PoolParams:
    """Square max-pooling window (frontend.py:68-80); pad < ksz so that no
    window lies wholly in padding."""

    ksz: int
    stride: int = 1
    pad: int = 0
    mode: str = "max"

    def __post_init__(self):
        if min(self.ksz, self.stride) < 1 or self.pad < 0:
            raise GraphError(f"bad pool params {self}")
        if self.pad >= self.ksz:
            raise GraphError(f"pool pad {self.pad} must be < window {self.ksz}")


@dataclass(frozen=True)
class ActParams:
    func: str = "relu"


@dataclass(frozen=True)
class ConvertParams:
    """Target layout of a Conversion node (frontend.py:88-90)."""

    target: DimsSpec


@dataclass(frozen=True)
class OpNode:
    name: str
    kind: str
    params: object
    inputs: tuple
    outputs: tuple
    fused_activation: str | None = None


@dataclass
class ComputeGraph:
    nodes: list = field(default_factory=list)
    edges: dict = field(default_factory=dict)
    sources: list = field(default_factory=list)
    sinks: list = field(default_factory=list)

    def node(self, name: str) -> OpNode:
        hit = [n for n in self.nodes if n.name == name]
        if not hit:
            raise GraphError(f"no node named '{name}'")
        return hit[0]

    def consumers_of(self, edge: str) -> list:
        return [n for n in self.nodes if edge in n.inputs]

    def producer_of(self, edge: str):
        hit = [n for n in self.nodes if edge in n.outputs]
        return hit[0] if hit else None

    def validate(self):
        """Single producer per edge, every read edge declared, acyclic (frontend.py:128-149)."""
        producers = {}
        for n in self.nodes:
            for e in n.outputs:
                if e in producers:
                    raise GraphError(f"edge '{e}' produced by both '{producers[e]}' and '{n.name}'")
                producers[e] = n.name
            for e in n.inputs:
                if e not in self.edges:
                    raise DanglingBottom(f"node '{n.name}' reads undeclared edge '{e}'")
        from .graphopt import schedule  # raises CycleDetected (a GraphError) on a cycle

        schedule(self)

    def recompute_endpoints(self):
        produced = {e for n in self.nodes if n.kind != KIND_INPUT for e in n.outputs}
        consumed = {e for n in self.nodes for e in n.inputs}
        self.sources = [e for e in self.edges if e not in produced]
        self.sinks = [e for e in self.edges if e not in consumed]

    def copy(self) -> "ComputeGraph":
        return ComputeGraph(list(self.nodes), dict(self.edges), list(self.sources), list(self.sinks))


def window_out(in_sz: int, ksz: int, stride: int, pad: int) -> int:
    """Output extent of a sliding window (frontend.py:441-442)."""
    return (in_sz + 2 * pad - ksz) // stride + 1


def conv_shapes(p: ConvParams, input_dims: DimsSpec, name: str = "conv"):
    """Filter, bias and output specs of one conv (infer_shapes conv branch, frontend.py:462-473)."""
    if input_dims.names != CANONICAL_DATA_DIMS:
        raise GraphError(f"input dims must be {CANONICAL_DATA_DIMS}, got {input_dims.names}")
    b, ic, h, w = input_dims.sizes
    oy, ox = window_out(h, p.ksz, p.stride, p.pad), window_out(w, p.ksz, p.stride, p.pad)
    if oy < 1:
        raise NonPositiveOutputDim(name, "y")
    if ox < 1:
        raise NonPositiveOutputDim(name, "x")
    filts = DimsSpec.row_major(CANONICAL_FILTS_DIMS, (p.out_chans, ic, p.ksz, p.ksz))
    bias = DimsSpec.row_major(CANONICAL_BIAS_DIMS, (p.out_chans,))
    out = DimsSpec.row_major(CANONICAL_DATA_DIMS, (b, p.out_chans, oy, ox))
    return filts, bias, out


def conv_graph(p: ConvParams, input_dims: DimsSpec, name: str = "conv") -> ComputeGraph:
    """Single-convolution graph, edges named as in frontend.py:523-532:
    ``data``, ``{name}_filts``, ``{name}_bias``, ``{name}_out``."""
    filts, bias, out = conv_shapes(p, input_dims, name)
    g = ComputeGraph()
    g.edges = {"data": input_dims, f"{name}_filts": filts, f"{name}_bias": bias, f"{name}_out": out}
    g.nodes = [
        OpNode("data_input", KIND_INPUT, None, (), ("data",)),
        OpNode(name, KIND_CONV, p, ("data", f"{name}_filts", f"{name}_bias"), (f"{name}_out",)),
    ]
    g.recompute_endpoints()
    return g


def set_fused_activation(node: OpNode, act: str | None) -> OpNode:
    return replace(node, fused_activation=act)


def with_fused(g: ComputeGraph, node_name: str, act: str | None) -> ComputeGraph:
    """Copy of ``g`` whose conv node carries ``fused_activation=act`` — the state
    graphopt.fuse_activations (graphopt.py:59-86) leaves a conv->ReLU pair in."""
    g2 = g.copy()
    g2.nodes = [replace(n, fused_activation=act) if n.name == node_name else n for n in g2.nodes]
    return g2


@dataclass(frozen=True)
class FlopCount:
    value: int
    exact: bool


def flops_of(node: OpNode, edges) -> FlopCount:
    """2*k^2*ic*oc*oy*ox*b; bias and activation excluded (frontend.py:499-514)."""
    if node.kind != KIND_CONV:
        return FlopCount(0, False)
    ind, out = edges[node.inputs[0]], edges[node.outputs[0]]
    if ind is None or out is None:
        raise GraphError(f"node '{node.name}': shapes not inferred")
    k = node.params.ksz
    value = 2 * k * k * ind.size_of("chan") * node.params.out_chans
    value *= out.size_of("y") * out.size_of("x") * out.size_of("img")
    return FlopCount(value, True)


def replace_node(g: ComputeGraph, old: str, new: OpNode) -> ComputeGraph:
    g = g.copy()
    g.nodes = [new if n.name == old else n for n in g.nodes]
    return g


# ----------------------------------------------------------------------------- shape inference


def infer_shapes(g: ComputeGraph, input_dims: DimsSpec) -> ComputeGraph:
    """Annotate every edge with its DimsSpec, walking the graph in schedule order
    from the Input node's edge (frontend.py:445-490)."""
    from .graphopt import schedule

    g = g.copy()
    for n in g.nodes:
        if n.kind == KIND_INPUT:
            if input_dims.names != CANONICAL_DATA_DIMS:
                raise GraphError(f"input dims must be {CANONICAL_DATA_DIMS}, got {input_dims.names}")
            g.edges[n.outputs[0]] = input_dims
    for name in schedule(g):
        n = g.node(name)
        if n.kind == KIND_INPUT:
            continue
        ind = g.edges[n.inputs[0]]
        if ind is None:
            raise GraphError(f"node '{n.name}': input edge not inferred")
        if n.kind == KIND_CONV:
            filts, bias, out = conv_shapes(n.params, ind, n.name)
            g.edges[n.inputs[1]], g.edges[n.inputs[2]], g.edges[n.outputs[0]] = filts, bias, out
        elif n.kind == KIND_POOL:
            b, c, h, w = (ind.size_of(d) for d in CANONICAL_DATA_DIMS)
            p = n.params
            oy, ox = window_out(h, p.ksz, p.stride, p.pad), window_out(w, p.ksz, p.stride, p.pad)
            if oy < 1:
                raise NonPositiveOutputDim(n.name, "y")
            if ox < 1:
                raise NonPositiveOutputDim(n.name, "x")
            g.edges[n.outputs[0]] = DimsSpec.row_major(CANONICAL_DATA_DIMS, (b, c, oy, ox))
        elif n.kind == KIND_ACT:
            g.edges[n.outputs[0]] = ind
        elif n.kind == KIND_CONVERT:
            g.edges[n.outputs[0]] = n.params.target
        else:
            raise GraphError(f"cannot infer shapes for kind {n.kind}")
    return g


# ----------------------------------------------------------------------------- network text

_TOKEN = re.compile(r"""
    (?P<nl>\n) | (?P<ws>[ \t\r]+) | (?P<comment>\#[^\n]*) |
    (?P<string>"[^"\n]*") | (?P<badstr>"[^"\n]*) |
    (?P<int>[0-9]+) | (?P<ident>[A-Za-z_][A-Za-z0-9_]*) | (?P<punct>[{}:]) | (?P<other>.)
""", re.X)

_LAYER_KINDS = {"Convolution": KIND_CONV, "Pooling": KIND_POOL, "ReLU": KIND_ACT}


def _lex(text: str):
    """(kind, text, line) tokens; kinds ident / string / int / punct, then eof."""
    out, line = [], 1
    for m in _TOKEN.finditer(text):
        k, v = m.lastgroup, m.group()
        if k == "nl":
            line += 1
        elif k in ("ws", "comment"):
            continue
        elif k == "badstr":
            raise NetSyntaxError(line, "closing quote")
        elif k == "other":
            raise NetSyntaxError(line, "token", v)
        else:
            out.append((k, v[1:-1] if k == "string" else v, line))
    out.append(("eof", "", line))
    return out


class _Cursor:
    def __init__(self, text: str):
        self.toks, self.i = _lex(text), 0

    @property
    def cur(self):
        return self.toks[self.i]

    def at(self, kind, text=None) -> bool:
        k, v, _ = self.cur
        return k == kind and (text is None or v == text)

    def expect(self, kind, text=None) -> str:
        k, v, line = self.cur
        if k != kind or (text is not None and v != text):
            raise NetSyntaxError(line, text if text is not None else kind, v)
        self.i += 1
        return v

    def field(self, allowed) -> str:
        line = self.cur[2]
        name = self.expect("ident")
        if name not in allowed:
            raise NetSyntaxError(line, f"one of {sorted(allowed)}", name)
        self.expect("punct", ":")
        return name

    def params(self, ints, enums=()):
        """``{ key: value ... }`` with each key at most once."""
        self.expect("punct", "{")
        got = {}
        while not self.at("punct", "}"):
            line = self.cur[2]
            key = self.field(set(ints) | set(enums))
            if key in got:
                raise NetSyntaxError(line, f"single '{key}'")
            got[key] = self.expect("ident") if key in enums else int(self.expect("int"))
        self.expect("punct", "}")
        return got

    def layer(self) -> dict:
        self.expect("punct", "{")
        lf = {"bottom": [], "top": []}
        while not self.at("punct", "}"):
            k, key, line = self.cur
            if k != "ident":
                raise NetSyntaxError(line, "layer field", key)
            self.i += 1
            if key in ("name", "type", "bottom", "top"):
                self.expect("punct", ":")
                val = self.expect("string")
                if key in ("bottom", "top"):
                    lf[key].append(val)
                elif key in lf:
                    raise NetSyntaxError(line, f"single '{key}' field")
                else:
                    lf[key] = val
            elif key == "convolution_param":
                got = self.params(("num_output", "kernel_size", "stride", "pad"))
                for req in ("num_output", "kernel_size"):
                    if req not in got:
                        raise NetSyntaxError(line, f"'{req}' in convolution_param")
                lf["conv"] = ConvParams(got["kernel_size"], got.get("stride", 1), got.get("pad", 0), got["num_output"])
            elif key == "pooling_param":
                got = self.params(("kernel_size", "stride", "pad"), ("pool",))
                if got.get("pool") != "MAX":
                    raise NetSyntaxError(line, "'pool: MAX'")
                if "kernel_size" not in got:
                    raise NetSyntaxError(line, "'kernel_size' in pooling_param")
                lf["pool"] = PoolParams(got["kernel_size"], got.get("stride", 1), got.get("pad", 0))
            else:
                raise NetSyntaxError(line, "supported layer field", key)
        self.expect("punct", "}")
        return lf


def parse_net(text: str) -> ComputeGraph:
    """Network text -> ComputeGraph (frontend.py:334-383): one node per layer in
    file order, ``{name}_filts`` / ``{name}_bias`` edges synthesised for each
    convolution, shapes inferred when the text carries input dims."""
    cur = _Cursor(text)
    g = ComputeGraph()
    input_dims = None
    if cur.at("ident", "input"):
        cur.expect("ident")
        cur.expect("punct", ":")
        src = cur.expect("string")
        dims = []
        for _ in range(4):
            cur.expect("ident", "input_dim")
            cur.expect("punct", ":")
            dims.append(int(cur.expect("int")))
        input_dims = DimsSpec.row_major(CANONICAL_DATA_DIMS, tuple(dims))
        g.edges[src] = None
        g.nodes.append(OpNode(f"{src}_input", KIND_INPUT, None, (), (src,)))
    while not cur.at("eof"):
        cur.expect("ident", "layer")
        lf = cur.layer()
        name, ltype = lf.get("name"), lf.get("type")
        if not isinstance(name, str):
            raise NetSyntaxError(0, "'name' field in every layer")
        if ltype not in _LAYER_KINDS:
            raise UnknownLayerType(f"layer '{name}': type {ltype!r} not supported")
        if len(lf["bottom"]) != 1 or len(lf["top"]) != 1:
            raise NetSyntaxError(0, f"layer '{name}': exactly one bottom and one top")
        bottom, top = lf["bottom"][0], lf["top"][0]
        if bottom == top:
            raise NetSyntaxError(0, f"layer '{name}': in-place layers (top == bottom) unsupported")
        if bottom not in g.edges:
            raise DanglingBottom(f"layer '{name}' reads undeclared edge '{bottom}'")
        if top in g.edges:
            raise GraphError(f"edge '{top}' produced twice")
        kind = _LAYER_KINDS[ltype]
        if kind == KIND_CONV:
            if "conv" not in lf:
                raise NetSyntaxError(0, f"layer '{name}': convolution_param required")
            ins, params = (bottom, f"{name}_filts", f"{name}_bias"), lf["conv"]
            g.edges[ins[1]] = g.edges[ins[2]] = None
        elif kind == KIND_POOL:
            if "pool" not in lf:
                raise NetSyntaxError(0, f"layer '{name}': pooling_param required")
            ins, params = (bottom,), lf["pool"]
        else:
            ins, params = (bottom,), ActParams("relu")
        g.edges[top] = None
        g.nodes.append(OpNode(name, kind, params, ins, (top,)))
    g.recompute_endpoints()
    g.validate()
    return infer_shapes(g, input_dims) if input_dims is not None else g


def pretty_print(g: ComputeGraph) -> str:
    """Canonical text of a parsed graph; parse_net(pretty_print(g)) reproduces g
    (frontend.py:386-434)."""
    out = []

    def block(n, ltype, param_name=None, fields=()):
        out.extend(["layer {", f'  name: "{n.name}"', f'  type: "{ltype}"', f'  bottom: "{n.inputs[0]}"',
                    f'  top: "{n.outputs[0]}"'])
        if param_name:
            out.append(f"  {param_name} {{")
            out.extend(f"    {k}: {v}" for k, v in fields)
            out.append("  }")
        out.append("}")

    for n in g.nodes:
        p = n.params
        if n.kind == KIND_INPUT:
            out.append(f'input: "{n.outputs[0]}"')
            spec = g.edges.get(n.outputs[0])
            if spec is not None:
                out.extend(f"input_dim: {s}" for s in spec.sizes)
        elif n.kind == KIND_CONV:
            block(n, "Convolution", "convolution_param",
                  (("num_output", p.out_chans), ("kernel_size", p.ksz), ("stride", p.stride), ("pad", p.pad)))
        elif n.kind == KIND_POOL:
            block(n, "Pooling", "pooling_param",
                  (("pool", "MAX"), ("kernel_size", p.ksz), ("stride", p.stride), ("pad", p.pad)))
        elif n.kind == KIND_ACT:
            block(n, "ReLU")
        else:
            raise GraphError(f"cannot pretty-print node kind {n.kind}")
    return "\n".join(out) + "\n"
