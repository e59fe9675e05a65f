"""CPU restatement of the reference's non-conv oracles (numpy) for the
whole-network path — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows the reference package:
* ``ref_pool_max``   cuclgen/oracle.py:100-116 — per-(img, chan) window max,
  out-of-range taps act as -inf (never win), float64 then cast to fp32.
  Restated as a max over the k*k strided tap views of a -inf-padded copy.
* ``ref_relu``       oracle.py:119-121 — np.maximum(x, 0) in fp32.
* ``convert_format`` ndarray.py:232-253 — permute named dims, then per dim crop
  (target smaller) or zero-pad at the end (target larger).
* ``check_node``     the per-node check of run_graph(check=True)
  (runner.py:230-244): node reference + compare at tolerance_for(ic*k*k).

Pinned against the reference's own outputs in tests/golden/net_cases.*
(made by tests/golden/make_net_golden.py, which imports cuclgen).
"""

from __future__ import annotations

import numpy as np

from .conv_ref import compare, ref_conv, tolerance_for


def ref_pool_max(x: np.ndarray, ksz: int, stride: int, pad: int) -> np.ndarray:
    x64 = np.asarray(x, dtype=np.float64)
    b, c, h, w = x64.shape
    oy, ox = (h + 2 * pad - ksz) // stride + 1, (w + 2 * pad - ksz) // stride + 1
    if oy < 1 or ox < 1:
        raise ValueError("non-positive output dims")
    xp = np.full((b, c, h + 2 * pad, w + 2 * pad), -np.inf)
    xp[:, :, pad:pad + h, pad:pad + w] = x64
    out = np.full((b, c, oy, ox), -np.inf)
    ys, xs = (oy - 1) * stride + 1, (ox - 1) * stride + 1
    for ky in range(ksz):
        for kx in range(ksz):
            np.maximum(out, xp[:, :, ky:ky + ys:stride, kx:kx + xs:stride], out=out)
    return out.astype(np.float32)


def ref_relu(x: np.ndarray) -> np.ndarray:
    return np.maximum(np.asarray(x, dtype=np.float32), np.float32(0.0))


def convert_format(x: np.ndarray, src_names, dst_names, dst_sizes) -> np.ndarray:
    if sorted(src_names) != sorted(dst_names):
        raise ValueError(f"cannot convert {src_names} to {dst_names}")
    a = np.transpose(np.asarray(x, dtype=np.float32), [list(src_names).index(n) for n in dst_names])
    out = np.zeros(tuple(dst_sizes), dtype=np.float32)
    common = tuple(slice(0, min(have, want)) for have, want in zip(a.shape, dst_sizes))
    out[common] = a[common]
    return out


def node_reference(node, edges, inputs: dict) -> np.ndarray:
    """CPU reference output of one node from canonical numpy inputs (runner.py:48-63)."""
    kind = node.kind
    if kind == "Convolution":
        x, f, b = (inputs[e] for e in node.inputs)
        p = node.params
        return ref_conv(x, f, b, p.stride, p.pad, relu=node.fused_activation == "relu")
    if kind == "Pooling":
        p = node.params
        return ref_pool_max(inputs[node.inputs[0]], p.ksz, p.stride, p.pad)
    if kind == "Activation":
        return ref_relu(inputs[node.inputs[0]])
    if kind == "Conversion":
        src, dst = edges[node.inputs[0]], edges[node.outputs[0]]
        return convert_format(inputs[node.inputs[0]], src.names, dst.names, dst.sizes)
    raise ValueError(f"no reference for kind {kind}")


def check_node(node, edges, inputs: dict, got):
    """The checker run_graph(check=...) calls: NdArray inputs / output in,
    CompareResult out, tolerance by the node's reduction length."""
    ins = {e: a.to_np() for e, a in inputs.items()}
    want = node_reference(node, edges, ins)
    terms = 1
    if node.kind == "Convolution":
        terms = edges[node.inputs[0]].size_of("chan") * node.params.ksz ** 2
    return compare(got.to_np(), want, tolerance_for(terms))
