"""fp8 mode (e4m3 operands, round to nearest, saturating, no scaling; fp32
accumulate on tcgen05 kind::f8f6f4) vs the CPU oracle.  Separately stated
tolerance:
* the reference's U[0.1, 1) data: |a-b| <= max(1e-6, 0.13 * max(|a|,|b|)),
  rigorous: every product carries <= 2*2^-4 + 2^-8 relative rounding (2^-4 per
  e4m3 operand) and all terms are positive; in practice errors of opposite sign
  cancel over the reduction, so the mean relative error is also checked (< 2e-2);
* signed U[-1, 1) data: |a-b| <= 0.13 * sum|x||w| + 1.1e-3 * sum(|x| + |w|) + 1e-6
  (the worst case per product: 2^-4 from each operand, plus 2^-10 absolute
  for values below the e4m3 subnormal range), ReLU clipping exactly where the
  oracle is below -bound.
The test also asserts the error is really fp8-sized (the mode cannot run fp32)."""

import numpy as np
import pytest

from oracle import conv_ref
from tests import golden_cases

pytestmark = pytest.mark.gpu

CASES, ARRAYS = golden_cases.load()
FP8_TOL = conv_ref.Tol(0.13)


def _run(g, x, f, b, params):
    import torch

    from paper_1611_06945_b200 import runner
    from paper_1611_06945_b200.variants import VARIANTS

    node = g.node("conv")
    vname = "conv_1x1" if node.params.ksz == 1 and node.params.pad == 0 else "conv_umma"
    if VARIANTS[vname].applies(node, g.edges, params) is not None:
        return None
    op = runner.ConvOp(VARIANTS[vname].generate(node, g.edges, params), *(torch.from_numpy(a).cuda() for a in (x, f, b)))
    op.y.fill_(float("nan"))
    op.launch()
    torch.cuda.synchronize()
    return op.y.cpu().numpy()


def _params():
    from paper_1611_06945_b200.variants import TuneParams

    return [TuneParams(bn=32, tma=1, prec=2), TuneParams(bn=64, split_k=2, tma=1, prec=2),
            TuneParams(bn=128, split_k=0, tma=1, prec=2), TuneParams(bn=64, tma=3, prec=2),
            TuneParams(bn=128, split_k=2, tma=3, prec=2), TuneParams(bn=64, tma=4, prec=2)]


def _graph(c, relu):
    from paper_1611_06945_b200.frontend import ConvParams, conv_graph, with_fused
    from paper_1611_06945_b200.ndarray import DimsSpec

    g = conv_graph(ConvParams(c["ksz"], c["stride"], c["pad"], c["out_chans"]), DimsSpec.row_major(("img", "chan", "y", "x"), c["in"]))
    return with_fused(g, "conv", "relu") if relu else g


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_fp8_golden_cases(cuda, case):
    g = _graph(case, case["act"] == "relu")
    x, f, b = golden_cases.inputs(case)
    want = conv_ref.ref_conv(x, f, b, case["stride"], case["pad"], relu=case["act"] == "relu")
    ran = 0
    for p in _params():
        got = _run(g, x, f, b, p)
        if got is None:
            continue
        res = conv_ref.compare(got, want, FP8_TOL)
        assert res.ok, (p.to_string(), res)
        mean_rel = float(np.mean(np.abs(got - want) / np.maximum(np.abs(want), 1e-6)))
        assert mean_rel < 2e-2, (p.to_string(), mean_rel)
        ran += 1
    c = case["in"][1]
    assert ran >= 1 or (c % 4 and c > 4)  # the TMA paths need 16-byte NHWC pixels (C % 4 == 0 or C <= 4)


def _abs_sum_bound(x, f, stride, pad):
    """sum over each output's window of (|x| + |w|)."""
    ones_w = np.ones_like(f)
    sx = conv_ref.ref_conv(np.abs(x), ones_w, np.zeros(f.shape[0], np.float32), stride, pad, relu=False)
    sw = np.abs(f).reshape(f.shape[0], -1).sum(1)[None, :, None, None]
    return sx.astype(np.float64) + sw


@pytest.mark.parametrize("row,batch,ptxt", [(34, 1, "BN=64,sk=1,tm=1"), (42, 5, "BN=128,sk=0,tm=1"),
                                            (38, 20, "BN=64,sk=2,tm=1"), (9, 20, "BN=64,sk=1,tm=3"),
                                            (41, 5, "BN=128,sk=1,tm=4"), (2, 1, "BN=32,sk=4,tm=1"),
                                            (34, 20, "BN=64,sk=1,tm=6"), (35, 5, "BN=128,sk=0,tm=6"),
                                            (33, 1, "BN=32,sk=2,tm=6")])
def test_fp8_signed_full_size(cuda, row, batch, ptxt):
    from paper_1611_06945_b200 import corpus
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.variants import TuneParams

    op = corpus.corpus(batch)[row]
    g = with_fused(op.graph(), "conv", "relu")
    p = TuneParams.from_string("MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1," + ptxt + ",pr=2")
    x, f, b = conv_ref.conv_inputs(op.batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz,
                                   f"fp8-signed:{row}:{batch}", low=-1.0, high=1.0)
    got = _run(g, x, f, b, p)
    assert got is not None
    got = got.astype(np.float64)
    pre = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=False).astype(np.float64)
    bound = 0.13 * conv_ref.signed_bound(x, f, op.stride, op.pad) + 1.1e-3 * _abs_sum_bound(x, f, op.stride, op.pad) + 1e-6
    err = np.abs(got - np.maximum(pre, 0.0))
    assert (err <= bound).all()
    must_clip = pre < -bound
    assert must_clip.any() and (got[must_clip] == 0.0).all()
    # really fp8: the error is far above fp32 rounding
    assert err.max() > 1e-3 * np.abs(pre).max()
