"""Winograd F(2x2,3x3) (conv_wino) at full size: every 3x3 / stride-1 op of the
sweep (14 corpus rows) at N = 1 / 5 / 20 against the float64 oracle.

* the reference's own data (U[0.1, 1), seed "wino:<row>:<N>") at the reference
  fp32 tolerance, unchanged (rel 1e-5 up to 4096 reduction terms,
  cuclgen/oracle.py:31-38): the transforms are exact-coefficient fp32 adds and
  the 16 GEMMs are fp32-exact 3xTF32, so no separate Winograd tolerance is needed;
* signed data (U[-1, 1)) at |a - b| <= 1e-5 * sum|x||w| + 1e-6 with ReLU
  required to clip exactly.
Both GEMM orientations (swap_ab 0: M stored [z][oc][p]; 1: [z][p][oc]) and the
split-K / stream-K fixups are exercised.
"""

import numpy as np
import pytest

from oracle import conv_ref

pytestmark = pytest.mark.gpu

PARAMS = ("BN=128,sk=1,sw=1,tm=1", "BN=64,sk=2,sw=0,tm=1", "BN=192,sk=0,sw=0,tm=1", "BN=128,sk=0,sw=1,tm=1")


def _ops():
    from paper_1611_06945_b200 import corpus

    out = []
    for row, op in corpus.sweep_ops([1, 5, 20]):
        if op.ksz == 3 and op.stride == 1:
            out.append(pytest.param(row, op, id=f"row{row:02d}-N{op.batch}"))
    return out


def _run(op, x, f, b, ptxt):
    import torch

    from paper_1611_06945_b200 import runner
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.variants import VARIANTS, TuneParams

    g = with_fused(op.graph(), "conv", "relu")
    node = g.node("conv")
    p = TuneParams.from_string("MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1," + ptxt)
    plan = VARIANTS["conv_wino"].generate(node, g.edges, p)
    cop = runner.ConvOp(plan, *(torch.from_numpy(a).cuda() for a in (x, f, b)))
    cop.y.fill_(float("nan"))
    cop.launch()
    torch.cuda.synchronize()
    return cop.y.cpu().numpy()


@pytest.mark.parametrize("row,op", _ops())
def test_wino_full_size_vs_oracle(cuda, row, op):
    assert op.pad <= 1
    ptxt = PARAMS[(row + op.batch) % len(PARAMS)]
    x, f, b = conv_ref.conv_inputs(op.batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz, f"wino:{row}:{op.batch}")
    got = _run(op, x, f, b, ptxt)
    want = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=True)
    res = conv_ref.compare(got, want, conv_ref.tolerance_for(op.in_chans * 9))
    assert res.ok, (ptxt, res)
    # signed data: cancellation-aware bound, exact clipping
    x, f, b = conv_ref.conv_inputs(op.batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz,
                                   f"wino-signed:{row}:{op.batch}", low=-1.0, high=1.0)
    got = _run(op, x, f, b, ptxt).astype(np.float64)
    pre = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=False).astype(np.float64)
    bound = 1e-5 * conv_ref.signed_bound(x, f, op.stride, op.pad) + 1e-6
    assert (np.abs(got - np.maximum(pre, 0.0)) <= bound).all(), ptxt
    must_clip = pre < -bound
    assert must_clip.any() and (got[must_clip] == 0.0).all()
