"""CPU restatement of the reference's conv oracle (numpy, float64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows cuclgen/oracle.py of the reference package:
* ``ref_conv``       oracle.py:69-99  — direct convolution, zero padding,
  float64 accumulation, bias added after the window sum, optional ReLU
  (np.maximum(., 0)), cast to fp32.  The reference loops over output
  positions and contracts each window with ``tensordot``; this restatement
  loops over the k*k filter taps and contracts channels with ``einsum`` —
  the same float64 sum, reassociated (tolerance-level identical; pinned
  against the reference's own outputs in tests/golden/).
* ``compare``        oracle.py:124-137 — |a-b| <= max(abs_floor, rel*max(|a|,|b|)).
* ``tolerance_for``  oracle.py:31-38  — rel 1e-5 for <= 4096 reduction terms, else 1e-3.
* ``seed_for`` / ``noise``  oracle.py:48-60 — sha256-seeded U[0.1, 1) fp32.

Parity is pinned (not "unpinned"): tests/test_oracle_golden.py checks this
module against golden vectors produced by importing the reference itself
(tests/golden/make_golden.py) and against the reference's known-answer
tests (tests/test_oracle.py in the reference: 7 = 3*2+1, identity kernel,
363-term window, linearity, zero filters).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

LONG_REDUCTION_TERMS = 4096


@dataclass(frozen=True)
class Tol:
    rel_tol: float = 1e-5
    abs_floor: float = 1e-6


def tolerance_for(reduction_terms: int) -> Tol:
    return Tol(1e-3) if reduction_terms > LONG_REDUCTION_TERMS else Tol()


def seed_for(signature: str) -> int:
    return int.from_bytes(hashlib.sha256(signature.encode()).digest()[:8], "little")


def noise(shape, seed: int, low: float = 0.1, high: float = 1.0) -> np.ndarray:
    n = int(np.prod(shape, dtype=np.int64))
    return np.random.default_rng(seed).uniform(low, high, size=n).astype(np.float32).reshape(shape)


def conv_inputs(b, ic, h, w, oc, ksz, seed: str, name: str = "conv", low=0.1, high=1.0):
    """The reference's synthetic operands for a single-conv graph: edges
    ``data``, ``{name}_filts``, ``{name}_bias`` seeded ``f"{seed}:{edge}"``
    (runner.py:39-45; edge names frontend.py:526-530)."""
    x = noise((b, ic, h, w), seed_for(f"{seed}:data"), low, high)
    f = noise((oc, ic, ksz, ksz), seed_for(f"{seed}:{name}_filts"), low, high)
    bias = noise((oc,), seed_for(f"{seed}:{name}_bias"), low, high)
    return x, f, bias


def ref_conv(x: np.ndarray, filts: np.ndarray, bias: np.ndarray, stride: int, pad: int, relu: bool = False) -> np.ndarray:
    """out[b,oc,oy,ox] = act(bias[oc] + sum_{ic,ky,kx} x_pad[b,ic,oy*s+ky,ox*s+kx] * f[oc,ic,ky,kx])."""
    x64 = np.asarray(x, dtype=np.float64)
    f64 = np.asarray(filts, dtype=np.float64)
    b, ic, h, w = x64.shape
    oc, fic, k, k2 = f64.shape
    if fic != ic or k != k2 or bias.shape != (oc,):
        raise ValueError("conv operand shapes inconsistent")
    oy = (h + 2 * pad - k) // stride + 1
    ox = (w + 2 * pad - k) // stride + 1
    if oy < 1 or ox < 1:
        raise ValueError("non-positive output dims")
    xp = np.zeros((b, ic, h + 2 * pad, w + 2 * pad), dtype=np.float64)
    xp[:, :, pad:pad + h, pad:pad + w] = x64
    acc = np.zeros((b, oc, oy, ox), dtype=np.float64)
    ys = (oy - 1) * stride + 1
    xs = (ox - 1) * stride + 1
    for ky in range(k):
        for kx in range(k):
            tap = xp[:, :, ky:ky + ys:stride, kx:kx + xs:stride]  # (b, ic, oy, ox)
            acc += np.einsum("bcyx,oc->boyx", tap, f64[:, :, ky, kx], optimize=True)
    acc += np.asarray(bias, dtype=np.float64)[None, :, None, None]
    if relu:
        acc = np.maximum(acc, 0.0)
    return acc.astype(np.float32)


@dataclass(frozen=True)
class CompareResult:
    ok: bool
    max_rel_err: float
    worst_index: tuple


def compare(a: np.ndarray, b: np.ndarray, tol: Tol = Tol()) -> CompareResult:
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {a.shape} vs {b.shape}")
    av, bv = a.astype(np.float64), b.astype(np.float64)
    diff = np.abs(av - bv)
    mag = np.maximum(np.abs(av), np.abs(bv))
    ok = bool(np.all(diff <= np.maximum(tol.abs_floor, tol.rel_tol * mag)))
    with np.errstate(invalid="ignore", divide="ignore"):
        rel = np.where(mag > 0, diff / mag, 0.0)
    if rel.size == 0:
        return CompareResult(ok, 0.0, ())
    worst = int(np.argmax(rel))
    return CompareResult(ok, float(rel.flat[worst]), tuple(int(i) for i in np.unravel_index(worst, a.shape)))


def signed_bound(x: np.ndarray, filts: np.ndarray, stride: int, pad: int) -> np.ndarray:
    """sum |x||w| per output: the error scale for signed-input
    suites, where cancellation makes pure relative error meaningless."""
    return ref_conv(np.abs(x), np.abs(filts), np.zeros(filts.shape[0], np.float32), stride, pad).astype(np.float64)
