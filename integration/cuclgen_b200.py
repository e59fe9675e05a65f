"""Reference-side binding: run the reference's (cuclgen 0.1.0) conv nodes on the B200.

This is the patch a maintainer of the reference would add, as a real module
(INTEGRATION.md describes it; tests/test_reference_dropin.py applies it to the
unmodified reference installed in baseline/_ref and runs the reference's own
entry points through it).  Pure ctypes + numpy, like the reference: no torch.

``install(cuclgen_pkg)`` patches a loaded ``cuclgen`` in place:

* ``cuclgen.runner.execute_node`` (runner.py:73-106, whose ``run_kernel`` call at
  :103 is the reference's device boundary, backend.py:1104-1133) runs conv
  nodes through ``b2c_conv_fwd_host`` (H2D of x / filters / bias, the kernel,
  D2H of y) and returns ``(canonical NdArray, CostReport(wall_ns=...))``; other
  node kinds keep the reference's simulator.  Every caller of ``execute_node``
  — ``validate_node`` (:109-115), ``tuner._evaluate`` (tuner.py:315),
  ``cli.cmd_bench`` (cli.py:97) and the reference's tests/helpers.py
  ``run_conv_variant`` (:59-79, when imported after ``install``) — is unchanged.
* The reference variants map onto the B200 kernels with their own knobs:
  ``conv_simple`` -> k_simple, ``conv_tiled`` -> k_tiled with the record's
  MNt / MNb / Kb / vw, ``conv_1x1`` / ``conv_fc`` -> the tcgen05 kernels.
* ``conv_umma``, ``conv_fc_stream`` and ``conv_wino`` (the B200-only variants the shipped
  TuneDBs name) are registered in ``cuclgen.variants.VARIANTS`` so that
  ``tuner.load_db`` (tuner.py:280 rejects unknown variant names) and
  ``select_variant`` (variants.py:840-856) accept the shipped B200 DBs.
* ``TuneParams.from_string`` (variants.py:73-91) keeps the B200 keys
  (``BN, sk, sw, dr, tm, oc, cl, pr``) in a ``TuneParams`` subclass instead of
  dropping them, so a DB record's tuned tile reaches the kernel verbatim.

The B200 variants have no CUCL text, so the reference's *model* objective
(static_cost_report over emitted source) cannot score them; on the B200 the
tuner times candidates on the device (paper_1611_06945_b200.tuner, objective
``wall``).
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, fields

_HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_LIB = os.path.join(os.path.dirname(_HERE), "paper_1611_06945_b200", "libb2conv.so")

VAR_ID = {"conv_simple": 0, "conv_tiled": 1, "conv_1x1": 2, "conv_fc": 3, "conv_umma": 4, "conv_fc_stream": 5,
          "conv_wino": 6}
B200_KEYS = ("BN", "sk", "sw", "dr", "tm", "oc", "cl", "pr")


class _Desc(ctypes.Structure):  # b2c_conv_desc (include/b2conv.h)
    _fields_ = [(n, ctypes.c_int32) for n in ("n", "c", "h", "w", "k", "r", "stride", "pad", "oh", "ow", "act", "prec")]


class _Tune(ctypes.Structure):  # b2c_tune (include/b2conv.h)
    _fields_ = [(n, ctypes.c_int32) for n in ("variant", "mnt0", "mnt1", "mnb0", "mnb1", "kb", "vw", "tile_n",
                                               "stages", "split_k", "swap_ab", "drain", "prepared", "tma", "cluster")]


class Binding:
    """libb2conv loaded with ctypes, plus one grow-only device scratch buffer."""

    def __init__(self, path: str | None = None):
        path = path or os.environ.get("B2CONV_LIB", DEFAULT_LIB)
        L = ctypes.CDLL(path)
        P, vp, sz = ctypes.POINTER, ctypes.c_void_p, ctypes.c_size_t
        L.b2c_conv_applies.argtypes = [P(_Desc), P(_Tune), ctypes.c_char_p, sz]
        L.b2c_conv_host_scratch.argtypes = [P(_Desc), P(_Tune)]
        L.b2c_conv_host_scratch.restype = sz
        L.b2c_conv_fwd_host.argtypes = [P(_Desc), P(_Tune), vp, vp, vp, vp, vp, sz, vp]
        L.b2c_device_alloc.argtypes = [sz]
        L.b2c_device_alloc.restype = vp
        L.b2c_device_free.argtypes = [vp]
        L.b2c_stream_synchronize.argtypes = [vp]
        L.b2c_last_error.restype = ctypes.c_char_p
        self.lib, self.path = L, path
        self._scratch, self._scratch_bytes = None, 0

    def error(self) -> str:
        return self.lib.b2c_last_error().decode(errors="replace")

    def applies(self, d: _Desc, t: _Tune) -> str | None:
        buf = ctypes.create_string_buffer(256)
        rc = self.lib.b2c_conv_applies(ctypes.byref(d), ctypes.byref(t), buf, 256)
        return None if rc == 0 else (buf.value.decode(errors="replace") or f"status {rc}")

    def scratch(self, nbytes: int):
        if nbytes > self._scratch_bytes:
            if self._scratch:
                self.lib.b2c_device_free(self._scratch)
            self._scratch = self.lib.b2c_device_alloc(nbytes)
            if not self._scratch:
                raise RuntimeError(f"b2c_device_alloc({nbytes}): {self.error()}")
            self._scratch_bytes = nbytes
        return self._scratch

    def fwd_host(self, d: _Desc, t: _Tune, x, w, b, y) -> int:
        """y = act(conv(x, w) + bias) on the device; returns device-synchronous wall ns."""
        need = self.lib.b2c_conv_host_scratch(ctypes.byref(d), ctypes.byref(t))
        scr = self.scratch(int(need))
        t0 = time.perf_counter_ns()
        rc = self.lib.b2c_conv_fwd_host(ctypes.byref(d), ctypes.byref(t), x.ctypes.data, w.ctypes.data,
                                        b.ctypes.data, y.ctypes.data, scr, self._scratch_bytes, None)
        if rc == 0:
            rc = self.lib.b2c_stream_synchronize(None)
        ns = time.perf_counter_ns() - t0
        if rc:
            raise RuntimeError(f"b2c_conv_fwd_host: {self.error()} (status {rc})")
        return ns


def _params_class(cuclgen):
    """TuneParams subclass carrying the B200 keys (string form as the shipped DBs write it)."""
    base = cuclgen.variants.TuneParams

    @dataclass(frozen=True)
    class B200TuneParams(base):
        bn: int = 128
        split_k: int = 1
        swap_ab: bool = False
        drain: int = 0
        tma: int = 1
        occ: int = 1
        cl: int = 1
        prec: int = 0

        def to_string(self) -> str:
            return (base.to_string(self) + f",BN={self.bn},sk={self.split_k},sw={int(self.swap_ab)},dr={self.drain}"
                    + (f",tm={self.tma}" if self.tma else "") + (f",oc={self.occ}" if self.occ != 1 else "")
                    + (f",cl={self.cl}" if self.cl != 1 else "") + (f",pr={self.prec}" if self.prec else ""))

    return B200TuneParams


def _conv_desc(cuclgen, node, edges, prec: int = 0) -> _Desc:
    b, ic, h, w = edges[node.inputs[0]].sizes
    _, oc, oy, ox = edges[node.outputs[0]].sizes
    p = node.params
    if node.fused_activation not in (None, "relu"):
        raise cuclgen.variants.Inapplicable(f"no fused form for activation '{node.fused_activation}'")
    return _Desc(b, ic, h, w, oc, p.ksz, p.stride, p.pad, oy, ox, 1 if node.fused_activation == "relu" else 0, prec)


def _tunes(variant: str, params) -> list:
    """b2c_tune candidates for a (variant, params) record, in preference order."""
    vid = VAR_ID[variant]
    base = dict(variant=vid, mnt0=params.mnt[0], mnt1=params.mnt[1], mnb0=params.mnb[0], mnb1=params.mnb[1],
                kb=params.kb, vw=params.vw, tile_n=128, stages=0, split_k=1, swap_ab=0, drain=0, prepared=0, tma=1,
                cluster=1)
    if hasattr(params, "bn"):  # a B200 record: its tuned tile verbatim
        base.update(tile_n=params.bn, split_k=params.split_k, swap_ab=int(params.swap_ab), drain=params.drain,
                    tma=params.tma, stages=params.occ if params.tma else 0, cluster=params.cl)
        return [_Tune(**base)]
    if vid in (0, 1, 5):
        return [_Tune(**base)]
    # a reference record (no B200 keys) for conv_1x1 / conv_fc: the TMA kernel's default tile,
    # then the swapped orientation, then the gather-fed kernel (any channel count)
    out = []
    for tma, swap in ((1, 0), (1, 1), (0, 0), (0, 1)):
        for bn in (128, 32):
            out.append(_Tune(**{**base, "tma": tma, "swap_ab": swap, "tile_n": bn}))
    return out


def install(cuclgen, lib_path: str | None = None) -> Binding:
    """Patch a loaded cuclgen package so its conv nodes run on the B200 (see module doc)."""
    import cuclgen.runner as R
    import cuclgen.variants as V

    if getattr(cuclgen, "_b200_binding", None) is not None:
        return cuclgen._b200_binding
    binding = Binding(lib_path)
    B200TuneParams = _params_class(cuclgen)
    orig_from_string = V.TuneParams.from_string
    base_names = {f.name for f in fields(V.TuneParams)}

    def from_string(text: str):
        kv = dict(part.partition("=")[::2] for part in text.split(","))
        p = orig_from_string(text)
        if not any(k in kv for k in B200_KEYS):
            return p
        try:
            extra = dict(bn=int(kv.get("BN", "128")), split_k=int(kv.get("sk", "1")), swap_ab=kv.get("sw", "0") == "1",
                         drain=int(kv.get("dr", "0")), tma=int(kv.get("tm", "0")), occ=int(kv.get("oc", "1")),
                         cl=int(kv.get("cl", "1")), prec=int(kv.get("pr", "0")))
        except ValueError as e:
            raise V.CuclgenError(f"bad tune-params string {text!r}: {e}") from None
        return B200TuneParams(**{n: getattr(p, n) for n in base_names}, **extra)

    V.TuneParams.from_string = staticmethod(from_string)

    def pick(node, edges, variant_name: str, params):
        prec = getattr(params, "prec", 0)
        d = _conv_desc(cuclgen, node, edges, prec)
        reasons = []
        for t in _tunes(variant_name, params):
            why = binding.applies(d, t)
            if why is None:
                return d, t
            reasons.append(why)
        raise V.Inapplicable(f"{variant_name} on '{node.name}': {reasons[0]}")

    class _B200Variant(V.Variant):
        kind = "Convolution"

        def applies(self, node, edges, params):
            r = V.Variant.applies(self, node, edges, params)
            if r:
                return r
            try:
                pick(node, edges, self.name, params)
            except V.Inapplicable as e:
                return str(e)
            return None

        def generate(self, node, edges, params, mode):
            raise V.Inapplicable(f"{self.name}: a B200 kernel (libb2conv), no CUCL source to instantiate")

    # Ranks tie with the reference's own variants and sort after them (insertion
    # order), so the reference's no-DB heuristic (variants.py:853-856) is unchanged;
    # the B200 variants are chosen by TuneDB records.
    class ConvUmma(_B200Variant):
        name, rank = "conv_umma", 1

    class ConvFCStream(_B200Variant):
        name, rank = "conv_fc_stream", 0

    class ConvWino(_B200Variant):
        name, rank = "conv_wino", 0

    V.VARIANTS.setdefault("conv_umma", ConvUmma())
    V.VARIANTS.setdefault("conv_fc_stream", ConvFCStream())
    V.VARIANTS.setdefault("conv_wino", ConvWino())

    orig_execute = R.execute_node

    def execute_node(node, edges, inputs, variant, params=V.DEFAULT_TUNE, mode="static", engine="vector",
                     thread_order=None, inst=None, src=None):
        if node.kind != "Convolution":
            return orig_execute(node, edges, inputs, variant, params, mode, engine, thread_order, inst, src)
        import numpy as np

        from cuclgen.backend import CostReport
        from cuclgen.ndarray import nda_from_np

        d, t = pick(node, edges, variant.name, params)
        x, w, b = (np.ascontiguousarray(inputs[e].to_np(), dtype=np.float32) for e in node.inputs)
        out = edges[node.outputs[0]]
        y = np.empty(tuple(out.sizes), np.float32)
        ns = binding.fwd_host(d, t, x, w, b, y)
        return nda_from_np(tuple(out.names), y), CostReport(wall_ns=ns)

    R.execute_node = execute_node
    cuclgen._b200_binding = binding
    return binding
