"""ctypes binding of libb2conv.so — the device boundary of the conv path.

This replaces the reference's simulated device (cuclgen/backend.py): where
runner.execute_node called ``run_kernel(ir, launch, buffers, ...)``
(backend.py:1104-1133, call site runner.py:103), the host now calls
``b2c_conv_fwd`` over device pointers (include/b2conv.h), and the
CostReport's ``wall_ns`` (backend.py:108) is CUDA-event device time.

PyTorch supplies only device memory and streams (``tensor.data_ptr()``,
``torch.cuda.current_stream().cuda_stream``); every FLOP runs in the
hand-written sm_100a kernels.  There is no CPU fallback: a missing library
or GPU raises.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

from .errors import CuclgenError, DeviceError, ExtensionMissing, Inapplicable, ShapeMismatch, Unsupported

LIB_NAME = "libb2conv.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

B2C_OK, B2C_INAPPLICABLE, B2C_BAD_ARGS, B2C_CUDA_ERROR, B2C_UNSUPPORTED = range(5)
VAR_SIMPLE, VAR_TILED, VAR_1X1, VAR_FC, VAR_UMMA, VAR_FC_STREAM, VAR_WINO = range(7)
PREC_FP32, PREC_BF16, PREC_FP8 = 0, 1, 2

# Every symbol include/b2conv.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "b2c_conv_applies",
    "b2c_conv_prepare",
    "b2c_conv_workspace",
    "b2c_conv_fwd",
    "b2c_conv_time",
    "b2c_conv_host_scratch",
    "b2c_conv_fwd_host",
    "b2c_conv_flops",
    "b2c_conv_bytes",
    "b2c_conv_launches",
    "b2c_conv_grid",
    "b2c_last_error",
    "b2c_version",
    "b2c_device_alloc",
    "b2c_device_free",
    "b2c_stream_synchronize",
    "b2c_pool_max_fwd",
    "b2c_relu_fwd",
    "b2c_xpose",
)

XPOSE_MAX_DIMS = 8


class ConvDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("n", "c", "h", "w", "k", "r", "stride", "pad", "oh", "ow", "act", "prec")]


class Tune(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "variant", "mnt0", "mnt1", "mnb0", "mnb1", "kb", "vw", "tile_n", "stages", "split_k", "swap_ab", "drain", "prepared", "tma", "cluster")]


class PoolDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("n", "c", "h", "w", "r", "stride", "pad", "oh", "ow")]


class XposeDesc(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("out_sizes", ctypes.c_int64 * XPOSE_MAX_DIMS),
                ("src_sizes", ctypes.c_int64 * XPOSE_MAX_DIMS),
                ("src_strides", ctypes.c_int64 * XPOSE_MAX_DIMS)]


_lib = None


def lib():
    """Load libb2conv.so once; raise ExtensionMissing if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(f"{LIB_PATH} is not built (run __graft_entry__.build())")
        try:
            L = ctypes.CDLL(LIB_PATH)
        except OSError as e:
            raise ExtensionMissing(f"cannot load {LIB_PATH}: {e}") from None
        P = ctypes.POINTER
        vp, sz = ctypes.c_void_p, ctypes.c_size_t
        L.b2c_conv_applies.argtypes = [P(ConvDesc), P(Tune), ctypes.c_char_p, sz]
        L.b2c_conv_prepare.argtypes = [P(ConvDesc), P(Tune), vp, vp, sz, vp]
        L.b2c_conv_workspace.argtypes = [P(ConvDesc), P(Tune)]
        L.b2c_conv_workspace.restype = sz
        L.b2c_conv_fwd.argtypes = [P(ConvDesc), P(Tune), vp, vp, vp, vp, vp, sz, vp]
        L.b2c_conv_time.argtypes = [P(ConvDesc), P(Tune), vp, vp, vp, vp, vp, sz, vp,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, P(ctypes.c_float)]
        L.b2c_conv_host_scratch.argtypes = [P(ConvDesc), P(Tune)]
        L.b2c_conv_host_scratch.restype = sz
        L.b2c_conv_fwd_host.argtypes = [P(ConvDesc), P(Tune), vp, vp, vp, vp, vp, sz, vp]
        L.b2c_conv_flops.argtypes = [P(ConvDesc)]
        L.b2c_conv_flops.restype = ctypes.c_int64
        L.b2c_conv_bytes.argtypes = [P(ConvDesc)]
        L.b2c_conv_bytes.restype = ctypes.c_int64
        L.b2c_conv_launches.argtypes = [P(ConvDesc), P(Tune)]
        L.b2c_conv_grid.argtypes = [P(ConvDesc), P(Tune)]
        L.b2c_pool_max_fwd.argtypes = [P(PoolDesc), vp, vp, vp]
        L.b2c_relu_fwd.argtypes = [vp, vp, ctypes.c_int64, vp]
        L.b2c_xpose.argtypes = [P(XposeDesc), vp, vp, vp]
        L.b2c_last_error.restype = ctypes.c_char_p
        L.b2c_version.restype = ctypes.c_char_p
        L.b2c_device_alloc.argtypes = [sz]
        L.b2c_device_alloc.restype = vp
        L.b2c_device_free.argtypes = [vp]
        L.b2c_stream_synchronize.argtypes = [vp]
        _lib = L
    return _lib


def check(rc: int, what: str = "b2conv"):
    """Map a C status to the reference's exception families (include/b2conv.h)."""
    if rc == B2C_OK:
        return
    msg = f"{what}: {lib().b2c_last_error().decode(errors='replace')}"
    if rc == B2C_INAPPLICABLE:
        raise Inapplicable(msg)
    if rc == B2C_BAD_ARGS:
        raise ShapeMismatch(msg)
    if rc == B2C_CUDA_ERROR:
        raise DeviceError(msg)
    if rc == B2C_UNSUPPORTED:
        raise Unsupported(msg)
    raise CuclgenError(f"{msg} (status {rc})")


def make_desc(b, ic, h, w, oc, ksz, stride, pad, oh, ow, relu: bool, prec: int = PREC_FP32) -> ConvDesc:
    return ConvDesc(b, ic, h, w, oc, ksz, stride, pad, oh, ow, 1 if relu else 0, prec)


def applies(desc: ConvDesc, tune: Tune) -> str | None:
    buf = ctypes.create_string_buffer(256)
    rc = lib().b2c_conv_applies(ctypes.byref(desc), ctypes.byref(tune), buf, 256)
    return None if rc == B2C_OK else (buf.value.decode() or f"status {rc}")


def workspace_bytes(desc: ConvDesc, tune: Tune) -> int:
    return int(lib().b2c_conv_workspace(ctypes.byref(desc), ctypes.byref(tune)))


def conv_flops(desc: ConvDesc) -> int:
    return int(lib().b2c_conv_flops(ctypes.byref(desc)))


def conv_bytes(desc: ConvDesc) -> int:
    return int(lib().b2c_conv_bytes(ctypes.byref(desc)))


def version() -> str:
    return lib().b2c_version().decode()


def _require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 conv path has no CPU fallback")
    return torch


def fwd(desc: ConvDesc, tune: Tune, x, w, bias, y, ws=None, stream=None):
    """Launch one conv on device tensors (torch CUDA fp32, contiguous). Async."""
    torch = _require_cuda()
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    ws_ptr, ws_len = (ws.data_ptr(), ws.numel() * ws.element_size()) if ws is not None else (None, 0)
    rc = lib().b2c_conv_fwd(ctypes.byref(desc), ctypes.byref(tune), x.data_ptr(), w.data_ptr(), bias.data_ptr(),
                            y.data_ptr(), ws_ptr, ws_len, st)
    check(rc, "b2c_conv_fwd")


def prepare(desc: ConvDesc, tune: Tune, w, ws, stream=None):
    """Pack the filters into the workspace (b2c_conv_prepare). Async."""
    torch = _require_cuda()
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    ws_ptr, ws_len = (ws.data_ptr(), ws.numel() * ws.element_size()) if ws is not None else (None, 0)
    check(lib().b2c_conv_prepare(ctypes.byref(desc), ctypes.byref(tune), w.data_ptr(), ws_ptr, ws_len, st),
          "b2c_conv_prepare")


def time_ms(desc: ConvDesc, tune: Tune, x, w, bias, y, ws=None, warmup=3, reps=10, l2_flush=True, stream=None) -> float:
    torch = _require_cuda()
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    ws_ptr, ws_len = (ws.data_ptr(), ws.numel() * ws.element_size()) if ws is not None else (None, 0)
    out = ctypes.c_float(0.0)
    rc = lib().b2c_conv_time(ctypes.byref(desc), ctypes.byref(tune), x.data_ptr(), w.data_ptr(), bias.data_ptr(),
                             y.data_ptr(), ws_ptr, ws_len, st, int(warmup), int(reps), 1 if l2_flush else 0,
                             ctypes.byref(out))
    check(rc, "b2c_conv_time")
    return float(out.value)


def _stream(stream):
    torch = _require_cuda()
    return stream if stream is not None else torch.cuda.current_stream().cuda_stream


def pool_max_fwd(desc: PoolDesc, x, y, stream=None):
    """Max pooling on device tensors (b2c_pool_max_fwd). Async."""
    st = _stream(stream)
    check(lib().b2c_pool_max_fwd(ctypes.byref(desc), x.data_ptr(), y.data_ptr(), st), "b2c_pool_max_fwd")


def relu_fwd(x, y, stream=None):
    """y = relu(x) over x.numel() fp32 elements (b2c_relu_fwd). Async."""
    st = _stream(stream)
    check(lib().b2c_relu_fwd(x.data_ptr(), y.data_ptr(), int(x.numel()), st), "b2c_relu_fwd")


def xpose_desc(src_names, src_sizes, src_strides, dst_names, dst_sizes) -> XposeDesc:
    """Descriptor of convert_format(src -> dst) for b2c_xpose: per output dim, the
    extent and element stride of the same-named source dim."""
    if set(src_names) != set(dst_names) or len(src_names) != len(dst_names):
        raise ShapeMismatch(f"cannot convert {tuple(src_names)} to {tuple(dst_names)}")
    if len(dst_names) > XPOSE_MAX_DIMS:
        raise Unsupported(f"{len(dst_names)} dims > {XPOSE_MAX_DIMS}")
    d = XposeDesc()
    d.ndim = len(dst_names)
    for i, name in enumerate(dst_names):
        j = list(src_names).index(name)
        d.out_sizes[i] = int(dst_sizes[i])
        d.src_sizes[i] = int(src_sizes[j])
        d.src_strides[i] = int(src_strides[j])
    return d


def xpose(desc: XposeDesc, x, y, stream=None):
    """Layout conversion on device tensors (b2c_xpose). Async."""
    st = _stream(stream)
    check(lib().b2c_xpose(ctypes.byref(desc), x.data_ptr(), y.data_ptr(), st), "b2c_xpose")


def alloc_workspace(desc: ConvDesc, tune: Tune, device=None):
    """Zero-filled device workspace (split-K partials + self-resetting tickets), or None."""
    torch = _require_cuda()
    n = workspace_bytes(desc, tune)
    if n == 0:
        return None
    return torch.zeros(n, dtype=torch.uint8, device=device or "cuda")


@dataclass
class CostReport:
    """Same fields as the reference CostReport (backend.py:101-116); on B200 the
    simulator counters are zero and ``wall_ns`` is CUDA-event device time."""

    alu_ops: int = 0
    global_loads: int = 0
    global_stores: int = 0
    local_loads: int = 0
    local_stores: int = 0
    barriers: int = 0
    wall_ns: int = 0

    def counters(self) -> tuple:
        return (self.alu_ops, self.global_loads, self.global_stores, self.local_loads, self.local_stores, self.barriers)
