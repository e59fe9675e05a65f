"""GPU parity: every variant through the C ABI vs the CPU oracle (and the
reference's own golden outputs), at the reference tolerance.

fp32 mode tolerance (stated): the reference rule verbatim —
|a-b| <= max(1e-6, rel*max(|a|,|b|)), rel = 1e-5 for ic*k*k <= 4096 else 1e-3
(cuclgen/oracle.py:31-38, :124-137).  Signed-input suite: |a-b| <= 1e-5 *
sum|x||w| + 1e-6, with ReLU required to clip exactly.
"""

import numpy as np
import pytest

from oracle import conv_ref
from tests import golden_cases

pytestmark = pytest.mark.gpu

CASES, ARRAYS = golden_cases.load()


def _graph(case_or_op, relu):
    from paper_1611_06945_b200.frontend import ConvParams, conv_graph, with_fused
    from paper_1611_06945_b200.ndarray import DimsSpec

    c = case_or_op
    p = ConvParams(ksz=c["ksz"], stride=c["stride"], pad=c["pad"], out_chans=c["out_chans"])
    g = conv_graph(p, DimsSpec.row_major(("img", "chan", "y", "x"), c["in"]))
    return with_fused(g, "conv", "relu") if relu else g


def _run_device(g, x, f, b, vname, params):
    import torch

    from paper_1611_06945_b200 import runner
    from paper_1611_06945_b200.variants import VARIANTS

    node = g.node("conv")
    plan = VARIANTS[vname].generate(node, g.edges, params)
    op = runner.ConvOp(plan, *(torch.from_numpy(a).cuda() for a in (x, f, b)))
    op.y.fill_(float("nan"))
    op.launch()
    torch.cuda.synchronize()
    return op.y.cpu().numpy()


def _variant_params(g):
    """(variant, params) pairs exercised on each case: every applicable variant,
    tcgen05 in both orientations and with split-K."""
    from paper_1611_06945_b200.variants import VARIANTS, TuneParams

    node = g.node("conv")
    out = [("conv_simple", TuneParams()), ("conv_tiled", TuneParams(mnt=(4, 4), mnb=(8, 8), kb=8, vw=4)),
           ("conv_tiled", TuneParams(mnt=(2, 2), mnb=(4, 4), kb=3, vw=2))]
    for v in ("conv_umma", "conv_1x1", "conv_fc"):
        for prm in (TuneParams(bn=32), TuneParams(bn=128, swap_ab=True), TuneParams(bn=64, split_k=2),
                    TuneParams(bn=32, tma=True), TuneParams(bn=128, swap_ab=True, tma=True),
                    TuneParams(bn=64, split_k=2, tma=True), TuneParams(bn=192, tma=True),
                    TuneParams(bn=96, swap_ab=True, split_k=3, tma=True), TuneParams(bn=64, tma=2),
                    TuneParams(bn=32, swap_ab=True, split_k=2, tma=2), TuneParams(bn=96, tma=2),
                    TuneParams(bn=32, split_k=2, tma=1), TuneParams(bn=64, split_k=0, tma=1),
                    TuneParams(bn=32, swap_ab=True, split_k=0, tma=1), TuneParams(bn=64, tma=1, occ=2),
                    TuneParams(bn=32, swap_ab=True, split_k=2, tma=1, occ=2), TuneParams(bn=64, tma=1, cl=2),
                    TuneParams(bn=96, split_k=2, tma=2, cl=2), TuneParams(bn=32, tma=3), TuneParams(bn=128, tma=3),
                    TuneParams(bn=16, swap_ab=True, split_k=2, tma=1), TuneParams(bn=16, swap_ab=True, split_k=0, tma=1),
                    TuneParams(bn=16, swap_ab=True, split_k=4, tma=2, occ=2),
                    TuneParams(bn=64, split_k=2, tma=3), TuneParams(bn=96, split_k=0, tma=3), TuneParams(bn=64, tma=3, occ=2),
                    TuneParams(bn=32, tma=4), TuneParams(bn=128, split_k=2, tma=4), TuneParams(bn=64, split_k=0, tma=4),
                    TuneParams(bn=64, tma=4, occ=2), TuneParams(bn=64, tma=1, cl=3),
                    TuneParams(bn=128, split_k=2, tma=1, cl=3), TuneParams(bn=192, tma=1, cl=3),
                    TuneParams(bn=128, tma=4, cl=3), TuneParams(bn=64, split_k=2, tma=3, cl=3),
                    TuneParams(bn=128, tma=3, cl=3), TuneParams(bn=128, split_k=0, tma=1, cl=3), TuneParams(bn=96, tma=1, cl=3),
                    TuneParams(bn=64, split_k=0, tma=4, cl=3), TuneParams(bn=32, split_k=2, tma=1, cl=4),
                    TuneParams(bn=64, split_k=4, tma=1, cl=4), TuneParams(bn=32, split_k=3, tma=3, cl=4),
                    TuneParams(bn=64, split_k=2, tma=4, cl=4), TuneParams(bn=32, swap_ab=True, split_k=4, tma=1, cl=4),
                    TuneParams(bn=96, tma=6), TuneParams(bn=64, split_k=2, tma=6), TuneParams(bn=96, tma=6, cl=3),
                    TuneParams(bn=128, split_k=0, tma=6)):
            out.append((v, prm))
    out += [("conv_wino", p) for p in (TuneParams(bn=64, tma=1), TuneParams(bn=128, split_k=2, tma=1),
                                       TuneParams(bn=192, split_k=0, tma=1), TuneParams(bn=64, swap_ab=True, tma=1),
                                       TuneParams(bn=128, swap_ab=True, split_k=0, tma=1))]
    out += [("conv_fc_stream", TuneParams(mnt=(1, 4), mnb=(8, 1), kb=1, vw=1)),
            ("conv_fc_stream", TuneParams(mnt=(1, 2), mnb=(4, 1), kb=1, vw=1)),
            ("conv_fc_stream", TuneParams(mnt=(1, 8), mnb=(2, 1), kb=1, vw=1)),
            ("conv_fc_stream", TuneParams(mnt=(1, 2), mnb=(8, 1), kb=2, vw=1)),
            ("conv_fc_stream", TuneParams(mnt=(1, 4), mnb=(4, 1), kb=2, vw=1)),
            ("conv_fc_stream", TuneParams(mnt=(1, 1), mnb=(8, 1), kb=2, vw=1))]
    return [(n, p) for n, p in out if VARIANTS[n].applies(node, g.edges, p) is None]


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_golden_cases_all_variants(cuda, case):
    g = _graph(case, case["act"] == "relu")
    x, f, b = golden_cases.inputs(case)
    want, step = golden_cases.expected(case, ARRAYS)
    tol = conv_ref.tolerance_for(case["reduction_terms"])
    checked = 0
    for vname, params in _variant_params(g):
        got = _run_device(g, x, f, b, vname, params)
        assert list(got.shape) == case["out_shape"]
        res = conv_ref.compare(got.reshape(-1)[::step], want, tol)
        assert res.ok, (vname, params.to_string(), res)
        checked += 1
    assert checked >= 3


def test_tiled_equals_simple_bit_exact(cuda):
    """Same fmaf sequence per output => identical bits (tests/test_variants.py:173-179)."""
    from paper_1611_06945_b200.variants import TuneParams

    case = {"ksz": 3, "stride": 1, "pad": 1, "out_chans": 5, "in": [2, 3, 6, 6]}
    g = _graph(case, False)
    x, f, b = conv_ref.conv_inputs(2, 3, 6, 6, 5, 3, "deg")
    s = _run_device(g, x, f, b, "conv_simple", TuneParams())
    for prm in (TuneParams(mnt=(1, 1), mnb=(1, 1), kb=1, vw=1), TuneParams(mnt=(4, 4), mnb=(8, 8), kb=8, vw=4),
                TuneParams(mnt=(8, 2), mnb=(4, 2), kb=5, vw=2)):
        t = _run_device(g, x, f, b, "conv_tiled", prm)
        assert np.array_equal(s, t), prm.to_string()


def _corpus_cases(batches):
    from paper_1611_06945_b200 import corpus

    out = []
    for bt in batches:
        for i, op in enumerate(corpus.corpus()):
            o = op.with_batch(bt)
            out.append(pytest.param(i, o, id=f"row{i:02d}-N{bt}"))
    return out


@pytest.mark.parametrize("row,op", _corpus_cases((1, 5, 20)))
def test_corpus_heuristic_variant_vs_oracle(cuda, row, op):
    """Every conv of the AlexNet/NiN/GoogLeNet sweep at N=1/5/20 with fused ReLU,
    on the variant select_variant picks (the shipped TuneDB when present)."""
    from paper_1611_06945_b200 import tuner
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.variants import select_variant
    import os

    g = with_fused(op.graph(), "conv", "relu")
    node = g.node("conv")
    db = tuner.load_db(tuner.shipped_db_path()) if os.path.exists(tuner.shipped_db_path()) else None
    v, params = select_variant(node, g.edges, db)
    x, f, b = conv_ref.conv_inputs(op.batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz,
                                   f"bench:{tuner.op_signature(node, g.edges)}")
    got = _run_device(g, x, f, b, v.name, params)
    want = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=True)
    res = conv_ref.compare(got, want, conv_ref.tolerance_for(op.in_chans * op.ksz ** 2))
    assert res.ok, (row, v.name, params.to_string(), res)


@pytest.mark.parametrize("vname", ["conv_simple", "conv_tiled", "conv_umma", "conv_umma_tma"])
def test_signed_inputs_relu_clips(cuda, vname):
    from paper_1611_06945_b200.variants import TuneParams

    case = {"ksz": 3, "stride": 1, "pad": 1, "out_chans": 48, "in": [2, 40, 14, 14]}
    g = _graph(case, True)
    x, f, b = conv_ref.conv_inputs(2, 40, 14, 14, 48, 3, "signed", low=-1.0, high=1.0)
    params = {"conv_simple": TuneParams(), "conv_tiled": TuneParams(mnt=(4, 4), mnb=(8, 8), kb=8, vw=4),
              "conv_umma": TuneParams(bn=64), "conv_umma_tma": TuneParams(bn=64, tma=True)}[vname]
    got = _run_device(g, x, f, b, vname.replace("_tma", ""), params)
    plain = conv_ref.ref_conv(x, f, b, 1, 1)
    want = np.maximum(plain, 0)
    bound = 1e-5 * conv_ref.signed_bound(x, f, 1, 1) + 1e-6
    assert np.all(np.abs(got.astype(np.float64) - want) <= bound)
    clipped = plain < -bound
    assert clipped.any() and np.all(got[clipped] == 0.0)


def test_split_k_deterministic(cuda):
    from paper_1611_06945_b200.variants import TuneParams

    case = {"ksz": 3, "stride": 1, "pad": 1, "out_chans": 256, "in": [1, 384, 13, 13]}
    g = _graph(case, True)
    x, f, b = conv_ref.conv_inputs(1, 384, 13, 13, 256, 3, "splitk")
    runs = [_run_device(g, x, f, b, "conv_umma", TuneParams(bn=128, split_k=8)) for _ in range(3)]
    assert all(np.array_equal(runs[0], r) for r in runs[1:])
    runs_t = [_run_device(g, x, f, b, "conv_umma", TuneParams(bn=128, split_k=8, tma=True)) for _ in range(3)]
    assert all(np.array_equal(runs_t[0], r) for r in runs_t[1:])
    want = conv_ref.ref_conv(x, f, b, 1, 1, relu=True)
    assert conv_ref.compare(runs[0], want, conv_ref.tolerance_for(384 * 9)).ok


def test_execute_node_and_host_e2e(cuda):
    """The public API: execute_node (host NdArrays in/out) and the C-ABI host call."""
    from paper_1611_06945_b200 import runner
    from paper_1611_06945_b200.variants import VARIANTS, TuneParams

    case = {"ksz": 5, "stride": 1, "pad": 2, "out_chans": 32, "in": [3, 16, 28, 28]}
    g = _graph(case, True)
    node = g.node("conv")
    inputs = runner.node_test_inputs(node, g.edges, "e2e")
    x, f, b = (inputs[e].to_np() for e in node.inputs)
    want = conv_ref.ref_conv(x, f, b, 1, 2, relu=True)
    got, rep = runner.execute_node(node, g.edges, inputs, VARIANTS["conv_umma"], TuneParams(bn=32))
    assert got.dims.names == ("img", "chan", "y", "x") and rep.wall_ns > 0
    assert conv_ref.compare(got.to_np(), want, conv_ref.tolerance_for(400)).ok
    plan = VARIANTS["conv_umma"].generate(node, g.edges, TuneParams(bn=32, split_k=2))
    hr = runner.HostRun.create(plan, x, f, b)
    hr.run()
    cuda.cuda.synchronize()
    assert np.array_equal(hr.hy.numpy(), got.to_np()) or conv_ref.compare(hr.hy.numpy(), want, conv_ref.tolerance_for(400)).ok


def test_sweep_on_device_and_db_roundtrip(cuda, tmp_path):
    from paper_1611_06945_b200 import tuner
    from paper_1611_06945_b200.variants import VARIANTS, select_variant

    case = {"ksz": 3, "stride": 1, "pad": 1, "out_chans": 64, "in": [1, 32, 14, 14]}
    g = _graph(case, True)
    node = g.node("conv")
    rec = tuner.sweep(node, g.edges, reps=3, warmup=1)
    assert rec.variant in VARIANTS and rec.objective == "wall" and rec.cost > 0
    db = tuner.TuneDB()
    db.add(rec)
    tuner.save_db(db, tmp_path / "db.tsv")
    db2 = tuner.load_db(tmp_path / "db.tsv")
    assert db2 == db
    v, params = select_variant(node, g.edges, db2)
    assert v.name == rec.variant and params == rec.params


def test_bad_args_raise(cuda):
    import torch

    from paper_1611_06945_b200 import backend
    from paper_1611_06945_b200.errors import ShapeMismatch

    d = backend.make_desc(1, 3, 8, 8, 4, 3, 1, 1, 7, 8, False)  # wrong oh
    t = backend.Tune(backend.VAR_SIMPLE, 1, 1, 1, 1, 1, 1, 32, 0, 1, 0, 0, 0, 0, 0)
    z = torch.zeros(1024, device="cuda")
    with pytest.raises(ShapeMismatch):
        backend.fwd(d, t, z, z, z, z)


@pytest.mark.parametrize("row,batch", [(25, 20), (13, 20), (25, 12), (13, 3), (13, 32)])
def test_fc_stream_staged_full_size(cuda, row, batch):
    """conv_fc_stream Kb=2 (x staged in smem) on AlexNet fc6 / fc7 at ragged and large batches."""
    from paper_1611_06945_b200 import corpus
    from paper_1611_06945_b200.variants import TuneParams

    op = corpus.corpus(batch)[row]
    c = {"ksz": op.ksz, "stride": op.stride, "pad": op.pad, "out_chans": op.out_chans,
         "in": (batch, op.in_chans, op.in_y, op.in_x)}
    g = _graph(c, True)
    x, f, b = conv_ref.conv_inputs(batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz, f"fcs:{row}:{batch}")
    want = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=True)
    tol = conv_ref.tolerance_for(op.in_chans * op.ksz ** 2)
    for p in (TuneParams(mnt=(1, 2), mnb=(8, 1), kb=2, vw=1), TuneParams(mnt=(1, 1), mnb=(4, 1), kb=2, vw=1)):
        got = _run_device(g, x, f, b, "conv_fc_stream", p)
        r = conv_ref.compare(got, want, tol)
        assert r.ok, (p.to_string(), r)


@pytest.mark.parametrize("row,batch,params", [(25, 5, "BN=16,sk=8,sw=1,dr=0,tm=1"), (13, 16, "BN=16,sk=4,sw=1,dr=0,tm=2,oc=2"),
                                              (25, 10, "BN=16,sk=0,sw=1,dr=0,tm=1"), (13, 3, "BN=16,sk=8,sw=1,dr=0,tm=1,oc=2")])
def test_fc_swap_bn16_full_size(cuda, row, batch, params):
    """conv_fc with the 16-image swapped tile (weights on M, N = 16): fc6 / fc7 at full size on
    reference data (fp32 tolerance) and signed data (exact ReLU clipping)."""
    from paper_1611_06945_b200 import corpus
    from paper_1611_06945_b200.variants import TuneParams

    op = corpus.corpus(batch)[row]
    c = {"ksz": op.ksz, "stride": op.stride, "pad": op.pad, "out_chans": op.out_chans,
         "in": (batch, op.in_chans, op.in_y, op.in_x)}
    g = _graph(c, True)
    p = TuneParams.from_string("MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1," + params)
    for low, high in ((0.1, 1.0), (-1.0, 1.0)):
        x, f, b = conv_ref.conv_inputs(batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz,
                                       f"fc16:{row}:{batch}:{low}", low=low, high=high)
        got = _run_device(g, x, f, b, "conv_fc", p)
        if low > 0:
            r = conv_ref.compare(got, conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=True),
                                 conv_ref.tolerance_for(op.in_chans * op.ksz ** 2))
            assert r.ok, r
        else:
            pre = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=False).astype(np.float64)
            bound = 1e-5 * conv_ref.signed_bound(x, f, op.stride, op.pad) + 1e-6
            assert (np.abs(got.astype(np.float64) - np.maximum(pre, 0.0)) <= bound).all()
            assert (got[pre < -bound] == 0.0).all() and (pre < -bound).any()


@pytest.mark.parametrize("row,batch", [(25, 1), (25, 5), (13, 5), (13, 8), (25, 3), (13, 7)])
def test_fc_bulk_full_size(cuda, row, batch):
    """conv_fc_stream Kb=3 (k_fc_bulk: weights + x streamed by TMA bulk copies through a
    shared-memory ring) on AlexNet fc6 / fc7: reference data at the fp32 tolerance, signed
    data with exact ReLU clipping, and bit-identical reruns (fixed reduction order)."""
    from paper_1611_06945_b200 import corpus
    from paper_1611_06945_b200.variants import TuneParams

    op = corpus.corpus(batch)[row]
    c = {"ksz": op.ksz, "stride": op.stride, "pad": op.pad, "out_chans": op.out_chans,
         "in": (batch, op.in_chans, op.in_y, op.in_x)}
    g = _graph(c, True)
    p = TuneParams(mnt=(1, 1), mnb=(8, 1), kb=3, vw=1)
    for low, high in ((0.1, 1.0), (-1.0, 1.0)):
        x, f, b = conv_ref.conv_inputs(batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz,
                                       f"fcb:{row}:{batch}:{low}", low=low, high=high)
        got = _run_device(g, x, f, b, "conv_fc_stream", p)
        if low > 0:
            r = conv_ref.compare(got, conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=True),
                                 conv_ref.tolerance_for(op.in_chans * op.ksz ** 2))
            assert r.ok, r
        else:
            pre = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=False).astype(np.float64)
            bound = 1e-5 * conv_ref.signed_bound(x, f, op.stride, op.pad) + 1e-6
            assert (np.abs(got.astype(np.float64) - np.maximum(pre, 0.0)) <= bound).all()
            assert (got[pre < -bound] == 0.0).all() and (pre < -bound).any()
            again = _run_device(g, x, f, b, "conv_fc_stream", p)
            assert np.array_equal(got, again)


@pytest.mark.parametrize("row,batch", [(0, 2), (29, 1), (31, 3), (39, 2), (41, 1)])
def test_direct_nchw_kxk_full_size(cuda, row, batch):
    """tm=4: k x k stride-1 convs read straight from NCHW by 4-D TMA boxes whose x start is
    rounded down to 16 bytes (the split warps apply the tap's shift): 28x28 / 56x56 GoogLeNet layers."""
    from paper_1611_06945_b200 import corpus
    from paper_1611_06945_b200.variants import VARIANTS, TuneParams

    op = corpus.corpus(batch)[row]
    c = {"ksz": op.ksz, "stride": op.stride, "pad": op.pad, "out_chans": op.out_chans,
         "in": (batch, op.in_chans, op.in_y, op.in_x)}
    g = _graph(c, True)
    x, f, b = conv_ref.conv_inputs(batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz, f"tm4:{row}", low=-1.0, high=1.0)
    want = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=True)
    bound = conv_ref.signed_bound(x, f, op.stride, op.pad)
    ran = 0
    for p in (TuneParams(bn=32, tma=4), TuneParams(bn=64, split_k=2, tma=4), TuneParams(bn=128, split_k=0, tma=4),
              TuneParams(bn=64, tma=4, occ=2), TuneParams(bn=64, tma=4, prec=1)):
        if VARIANTS["conv_umma"].applies(g.node("conv"), g.edges, p) is not None:
            continue
        got = _run_device(g, x, f, b, "conv_umma", p)
        err = np.abs(got.astype(np.float64) - want.astype(np.float64))
        k = 8e-3 if p.prec else 1e-5
        assert (err <= k * bound + 1e-6).all(), (p.to_string(), float((err / (bound + 1e-30)).max()))
        ran += 1
    assert ran >= 4


def test_split_k_ops_concurrent_on_streams(cuda):
    """Split-K / stream-K launches of several ops overlapping on three streams give
    the same bits as serial launches (the fixup never waits on another CTA, so
    concurrent grids cannot deadlock it)."""
    import torch

    from paper_1611_06945_b200 import corpus, runner
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.variants import VARIANTS, TuneParams

    ops = []
    for row, batch, p in ((40, 5, TuneParams(bn=96, split_k=4, tma=1)), (42, 5, TuneParams(bn=128, split_k=0, tma=1)),
                          (36, 1, TuneParams(bn=32, split_k=8, swap_ab=True, tma=1)), (37, 5, TuneParams(bn=64, split_k=0, tma=1)),
                          (2, 5, TuneParams(bn=32, split_k=4, tma=2)), (38, 1, TuneParams(bn=32, split_k=4, tma=1))):
        op = corpus.corpus(batch)[row]
        g = with_fused(op.graph(), "conv", "relu")
        node = g.node("conv")
        inputs = runner.node_test_inputs(node, g.edges, f"conc:{row}")
        x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
        ops.append(runner.ConvOp(VARIANTS["conv_umma" if op.ksz > 1 else "conv_1x1"].generate(node, g.edges, p), x, w, b))
    ref = []
    for o in ops:
        o.launch()
        torch.cuda.synchronize()
        ref.append(o.y.clone())
    streams = [torch.cuda.Stream() for _ in range(3)]
    for _ in range(5):
        for i, o in enumerate(ops):
            o.launch(streams[i % 3].cuda_stream)
    torch.cuda.synchronize()
    for o, r in zip(ops, ref):
        assert torch.equal(o.y, r)


@pytest.mark.parametrize("row,params", [(38, "BN=96,sk=4,sw=0,dr=0,tm=1"), (2, "BN=32,sk=2,sw=0,dr=0,tm=2"),
                                        (41, "BN=64,sk=1,sw=0,dr=0,tm=4"), (25, "BN=32,sk=4,sw=1,dr=0,tm=1")])
def test_batch_slabs_concatenate_bit_identical(cuda, row, params):
    """batch sharding = contiguous image slabs (shard.batch_slab); with the same
    kernel choice, running the slabs separately and concatenating gives the single-run bits."""
    import torch

    from paper_1611_06945_b200 import corpus, runner, shard
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.variants import VARIANTS, TuneParams

    p = TuneParams.from_string("MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1," + params)
    n = 8
    full = corpus.corpus(n)[row]
    g = with_fused(full.graph(), "conv", "relu")
    node = g.node("conv")
    inputs = runner.node_test_inputs(node, g.edges, f"slab:{row}")
    x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
    vname = "conv_fc" if row == 25 else ("conv_1x1" if full.ksz == 1 else "conv_umma")
    whole = runner.ConvOp(VARIANTS[vname].generate(node, g.edges, p), x, w, b)
    whole.launch()
    parts = []
    for rank in range(3):
        start, count = shard.batch_slab(n, 3, rank)
        op = full.with_batch(count)
        gs = with_fused(op.graph(), "conv", "relu")
        o = runner.ConvOp(VARIANTS[vname].generate(gs.node("conv"), gs.edges, p), x[start:start + count].contiguous(), w, b)
        o.launch()
        parts.append(o.y)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, 0), whole.y)


@pytest.mark.parametrize("row,batch,params", [(34, 20, "BN=96,sk=1,sw=0,dr=0,tm=6"), (33, 5, "BN=96,sk=1,sw=0,dr=0,tm=6,cl=3"),
                                              (35, 20, "BN=64,sk=1,sw=0,dr=0,tm=6"), (34, 1, "BN=32,sk=4,sw=0,dr=0,tm=6"),
                                              (35, 5, "BN=64,sk=0,sw=0,dr=0,tm=6")])
def test_first_layer_space_to_depth_full_size(cuda, row, batch, params):
    """tma=6: AlexNet / NiN / GoogLeNet conv1 as R'xR' stride-1 convs over a space-to-depth copy of x
    (C*S*S channels, re-arranged filters): same fp32-exact products, so the reference tolerance holds;
    also on signed data with exact ReLU clipping."""
    import torch

    from paper_1611_06945_b200 import corpus, runner
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.variants import VARIANTS, TuneParams

    op = corpus.corpus(batch)[row]
    g = with_fused(op.graph(), "conv", "relu")
    node = g.node("conv")
    p = TuneParams.from_string("MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1," + params)
    plan = VARIANTS["conv_umma"].generate(node, g.edges, p)
    for low, high in ((0.1, 1.0), (-1.0, 1.0)):
        x, f, b = conv_ref.conv_inputs(op.batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz,
                                       f"s2d:{row}:{batch}:{low}", low=low, high=high)
        cop = runner.ConvOp(plan, *(torch.from_numpy(a).cuda() for a in (x, f, b)))
        cop.y.fill_(float("nan"))
        cop.launch()
        torch.cuda.synchronize()
        got = cop.y.cpu().numpy()
        if low > 0:
            want = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=True)
            res = conv_ref.compare(got, want, conv_ref.tolerance_for(op.in_chans * op.ksz * op.ksz))
            assert res.ok, res
        else:
            pre = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=False).astype(np.float64)
            bound = 1e-5 * conv_ref.signed_bound(x, f, op.stride, op.pad) + 1e-6
            assert (np.abs(got.astype(np.float64) - np.maximum(pre, 0.0)) <= bound).all()
            assert (got[pre < -bound] == 0.0).all()
