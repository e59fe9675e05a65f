"""bf16 mode (bf16 operands, fp32 accumulate) of the TMA tcgen05 kernel vs the
CPU oracle.  Separately stated tolerance: on the reference's
U[0.1, 1) inputs |a-b| <= max(1e-6, 4e-3 * max(|a|,|b|)); on signed inputs
|a-b| <= 8e-3 * sum|x||w| + 1e-6 (each product carries at most 2^-9 rounding
from each bf16 operand), with ReLU clipping exactly where the oracle clips."""

import numpy as np
import pytest

from oracle import conv_ref
from tests import golden_cases

pytestmark = pytest.mark.gpu

CASES, ARRAYS = golden_cases.load()
BF16_TOL = conv_ref.Tol(4e-3)


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

    return [TuneParams(bn=32, tma=1, prec=1), TuneParams(bn=64, split_k=2, tma=1, prec=1),
            TuneParams(bn=128, tma=2, prec=1), TuneParams(bn=192, split_k=0, tma=1, prec=1),
            TuneParams(bn=64, split_k=0, tma=2, prec=1), TuneParams(bn=64, tma=3, prec=1),
            TuneParams(bn=128, split_k=2, tma=3, prec=1), TuneParams(bn=64, tma=5, prec=1),
            TuneParams(bn=128, split_k=2, tma=5, prec=1), TuneParams(bn=192, split_k=0, tma=5, prec=1),
            TuneParams(bn=128, tma=5, cl=3, prec=1), TuneParams(bn=192, split_k=2, tma=5, cl=3, prec=1),
            TuneParams(bn=128, split_k=0, tma=5, cl=3, prec=1), TuneParams(bn=64, split_k=1, tma=6, prec=1)]


def _graph(c, relu):
    from paper_1611_06945_b200.frontend import ConvParams, conv_graph, with_fused
    from paper_1611_06945_b200.ndarray import DimsSpec

    g = conv_graph(ConvParams(c["ksz"], c["stride"], c["pad"], c["out_chans"]), DimsSpec.row_major(("img", "chan", "y", "x"), c["in"]))
    return with_fused(g, "conv", "relu") if relu else g


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_bf16_golden_cases(cuda, case):
    g = _graph(case, case["act"] == "relu")
    x, f, b = golden_cases.inputs(case)
    want = conv_ref.ref_conv(x, f, b, case["stride"], case["pad"], relu=case["act"] == "relu")
    ran = 0
    for p in _params():
        got = _run(g, x, f, b, p)
        if got is None:
            continue
        ran += 1
        r = conv_ref.compare(got, want, BF16_TOL)
        assert r.ok, (p.to_string(), r)
    if case["in"][1] % 4 == 0 or case["in"][1] <= 4:
        assert ran > 0


@pytest.mark.parametrize("row,batch", [(42, 20), (34, 5), (2, 20), (40, 5), (35, 1), (20, 5), (33, 20), (35, 20)])
def test_bf16_full_size_signed(cuda, row, batch):
    from paper_1611_06945_b200 import corpus
    from paper_1611_06945_b200.variants import TuneParams

    op = corpus.corpus(batch)[row]
    c = {"ksz": op.ksz, "stride": op.stride, "pad": op.pad, "out_chans": op.out_chans,
         "in": (batch, op.in_chans, op.in_y, op.in_x)}
    g = _graph(c, True)
    x, f, b = conv_ref.conv_inputs(batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz, f"bf16:{row}", low=-1.0, high=1.0)
    want = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=True)
    bound = conv_ref.signed_bound(x, f, op.stride, op.pad)
    for p in (TuneParams(bn=64, tma=1, prec=1), TuneParams(bn=128, split_k=0, tma=1, prec=1),
              TuneParams(bn=128, split_k=0, tma=5, prec=1), TuneParams(bn=192, split_k=0, tma=5, cl=3, prec=1),
              TuneParams(bn=64, split_k=1, tma=6, prec=1), TuneParams(bn=128, split_k=0, tma=6, prec=1)):
        got = _run(g, x, f, b, p)
        if got is None and p.tma == 5:  # the bf16-NHWC SS path needs in_chans % 8 == 0 (not first layers)
            assert op.in_chans % 8 or op.in_chans <= 4
            continue
        if got is None and p.tma == 6:  # space-to-depth: strided first layers only
            assert op.in_chans > 4 or op.stride == 1
            continue
        assert got is not None
        err = np.abs(got.astype(np.float64) - want.astype(np.float64))
        assert (err <= 8e-3 * bound + 1e-6).all(), (p.to_string(), float((err / (bound + 1e-30)).max()))
        assert (got >= 0).all() and (got == 0).any()  # ReLU clipped (signed data)
        # and it really is bf16 arithmetic: errors far above the fp32-exact path's ~1e-7 of the bound
        assert float((err / (bound + 1e-30)).max()) > 1e-5


def test_bf16_applicability(cuda):
    from paper_1611_06945_b200 import corpus
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.variants import VARIANTS, TuneParams

    op = corpus.corpus(5)[42]
    g = with_fused(op.graph(), "conv", "relu")
    node = g.node("conv")
    assert VARIANTS["conv_umma"].applies(node, g.edges, TuneParams(bn=64, tma=1, prec=1)) is None
    assert VARIANTS["conv_umma"].applies(node, g.edges, TuneParams(bn=64, tma=0, prec=1)) is not None  # gather kernel
    assert VARIANTS["conv_umma"].applies(node, g.edges, TuneParams(bn=64, tma=1, swap_ab=True, prec=1)) is not None
    assert VARIANTS["conv_tiled"].applies(node, g.edges, TuneParams(prec=1)) is not None
