"""Op description: the conv-node types of the reference front end.

Only the part of the reference's L1 layer that lies on the conv path is
mirrored: ConvParams (cuclgen/frontend.py:56-65), OpNode (:93-100),
ComputeGraph (:103-159), window_out (:441-442), the conv branch of
infer_shapes (:445-490), flops_of (:499-514) and conv_graph (:523-532).
The layer-block network parser (frontend.py:166-434) is not on the per-op
conv path and is out of scope.
"""

from __future__ import annotations

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
class ActParams:
    func: str = "relu"


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
