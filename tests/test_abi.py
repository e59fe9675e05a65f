"""The C-ABI library loads on CPU and exports every symbol include/b2conv.h declares;
host-side entry points that need no GPU behave (applicability, sizing, errors)."""

import ctypes
import os
import re

import pytest

from paper_1611_06945_b200 import backend

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "b2conv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(b2c_[a-z_0-9]+)\s*\(", src)))


def test_header_matches_binding_table():
    assert declared_functions() == sorted(backend.EXPORTS)


def test_library_exports_all_symbols():
    lib = backend.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_version():
    assert backend.version().startswith("b2conv ") and "sm_100a" in backend.version()


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", backend.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def _desc(**kw):
    d = dict(b=1, ic=3, h=227, w=227, oc=96, ksz=11, stride=4, pad=0, oh=55, ow=55, relu=True)
    d.update(kw)
    return backend.make_desc(d["b"], d["ic"], d["h"], d["w"], d["oc"], d["ksz"], d["stride"], d["pad"], d["oh"], d["ow"], d["relu"])


def _tune(variant, **kw):
    t = dict(mnt0=4, mnt1=4, mnb0=16, mnb1=16, kb=4, vw=4, tile_n=128, stages=0, split_k=1, swap_ab=0, drain=0, prepared=0, tma=0, cluster=0)
    t.update(kw)
    return backend.Tune(variant, *t.values())


def test_applicability_reasons():
    d = _desc()
    assert backend.applies(d, _tune(backend.VAR_SIMPLE)) is None
    assert backend.applies(d, _tune(backend.VAR_UMMA, tile_n=96)) is None
    assert "kernel size" in backend.applies(d, _tune(backend.VAR_1X1))
    assert "whole input" in backend.applies(d, _tune(backend.VAR_FC))
    assert "tile_n" in backend.applies(d, _tune(backend.VAR_UMMA, tile_n=100))
    assert "1024" in backend.applies(d, _tune(backend.VAR_TILED, mnb0=64, mnb1=32))
    assert "output channels" in backend.applies(_desc(oc=2), _tune(backend.VAR_TILED))
    assert backend.applies(d, _tune(backend.VAR_UMMA, tile_n=96, tma=1)) is None  # first layer: x-window TMA path
    assert "swap_ab=0" in backend.applies(d, _tune(backend.VAR_UMMA, tile_n=96, tma=1, swap_ab=1))
    assert "in_chans % 4" in backend.applies(_desc(ic=6), _tune(backend.VAR_UMMA, tile_n=96, tma=1))
    assert backend.applies(_desc(ic=64), _tune(backend.VAR_UMMA, tile_n=96, tma=1)) is None
    fc = _desc(b=5, ic=256, h=6, w=6, oc=4096, ksz=6, stride=1, pad=0, oh=1, ow=1)
    assert backend.applies(fc, _tune(backend.VAR_FC, tile_n=32, swap_ab=1, split_k=4, tma=1)) is None
    assert backend.applies(fc, _tune(backend.VAR_FC, tile_n=32, swap_ab=1, split_k=8)) is None


def test_launch_counts():
    d = _desc()
    lib = backend.lib()
    assert lib.b2c_conv_launches(ctypes.byref(d), ctypes.byref(_tune(backend.VAR_UMMA, tile_n=96))) == 2
    assert lib.b2c_conv_launches(ctypes.byref(d), ctypes.byref(_tune(backend.VAR_UMMA, tile_n=96, prepared=1))) == 1
    assert lib.b2c_conv_launches(ctypes.byref(d), ctypes.byref(_tune(backend.VAR_SIMPLE))) == 1


def test_bad_descriptor_is_rejected():
    assert "inconsistent" in backend.applies(_desc(oh=54), _tune(backend.VAR_SIMPLE))
    assert backend.applies(_desc(stride=0), _tune(backend.VAR_SIMPLE))


def test_workspace_and_work_accounting():
    d = _desc()
    kblocks = -(-363 // 32)  # C = 3 < 32: flat K order
    packed = 1 * kblocks * 2 * 96 * 32 * 4  # one 96-row filter tile, raw + lo
    assert backend.workspace_bytes(d, _tune(backend.VAR_SIMPLE)) == 0
    assert backend.workspace_bytes(d, _tune(backend.VAR_UMMA, tile_n=96)) >= packed
    ws = backend.workspace_bytes(d, _tune(backend.VAR_UMMA, tile_n=96, split_k=4))
    tiles = -(-3025 // 128)
    assert ws >= packed + tiles * 4 * 96 * 128 * 4 + tiles * 4
    assert backend.conv_flops(d) == 210_830_400
    assert backend.conv_bytes(d) == 1_919_724


def test_product_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1611_06945_b200 import runner
    from paper_1611_06945_b200.errors import DeviceError
    from paper_1611_06945_b200.frontend import ConvParams, conv_graph
    from paper_1611_06945_b200.ndarray import DimsSpec
    from paper_1611_06945_b200.variants import VARIANTS

    g = conv_graph(ConvParams(ksz=3, pad=1, out_chans=4), DimsSpec.row_major(("img", "chan", "y", "x"), (1, 2, 5, 5)))
    node = g.node("conv")
    inputs = runner.node_test_inputs(node, g.edges, "x")
    with pytest.raises(DeviceError):
        runner.execute_node(node, g.edges, inputs, VARIANTS["conv_simple"])
