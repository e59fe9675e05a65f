"""Host-side mirror of the reference interface: op description, corpus, variant
API and TuneDB contract (restating the reference's own tests where they apply:
pkg/tests/test_frontend.py, test_variants.py:327-360, test_tuner.py)."""

import threading

import numpy as np
import pytest

from paper_1611_06945_b200 import corpus, tuner
from paper_1611_06945_b200.backend import CostReport
from paper_1611_06945_b200.errors import CuclgenError, Inapplicable
from paper_1611_06945_b200.frontend import ConvParams, conv_graph, flops_of, window_out, with_fused
from paper_1611_06945_b200.ndarray import DimsSpec, convert_format, dims_check, make_nda, nda_from_np
from paper_1611_06945_b200.variants import (DEFAULT_TUNE, VARIANTS, TuneParams, select_variant,
                                            variants_for_kind)

NCHW = ("img", "chan", "y", "x")


def g_of(ksz, stride, pad, oc, dims):
    return conv_graph(ConvParams(ksz=ksz, stride=stride, pad=pad, out_chans=oc), DimsSpec.row_major(NCHW, dims))


def test_window_out_cases():
    assert window_out(227, 11, 4, 0) == 55
    assert window_out(224, 7, 2, 3) == 112
    assert window_out(13, 3, 1, 1) == 13
    assert window_out(6, 6, 1, 0) == 1


def test_flops_known_values():
    g = g_of(5, 1, 2, 32, (5, 16, 28, 28))
    assert flops_of(g.node("conv"), g.edges).value == 100_352_000
    g = g_of(6, 1, 0, 4096, (5, 256, 6, 6))
    assert flops_of(g.node("conv"), g.edges).value == 377_487_360


def test_conv_graph_edges_and_shapes():
    g = g_of(11, 4, 0, 96, (1, 3, 227, 227))
    assert set(g.edges) == {"data", "conv_filts", "conv_bias", "conv_out"}
    assert g.edges["conv_filts"].sizes == (96, 3, 11, 11)
    assert g.edges["conv_out"].sizes == (1, 96, 55, 55)
    assert g.sources == ["data", "conv_filts", "conv_bias"] and g.sinks == ["conv_out"]
    with pytest.raises(CuclgenError):
        ConvParams(ksz=0)


def test_corpus_rows_and_gate():
    ops = corpus.corpus()
    assert len(ops) == 43
    assert corpus.corpus_gate(ops) == []
    assert all(op.flops_published_consistent for op in ops)
    assert ops[34].conv_params == ConvParams(ksz=11, stride=4, pad=0, out_chans=96)
    assert [op.pad for op in ops[:3]] == [2, 2, 0]
    assert ops[25].flops_computed == 377_487_360
    total = sum(op.flops_computed for op in ops)
    assert total == pytest.approx(2.936e10, rel=1e-3)
    assert [o.batch for o in corpus.corpus(20)] == [20] * 43
    assert corpus.corpus(20)[34].flops_computed == 4 * ops[34].flops_computed


def test_corpus_csv_roundtrip_and_shipped_file():
    ops = corpus.corpus()
    assert corpus.from_csv(corpus.to_csv(ops)) == ops
    assert corpus.load_corpus(corpus.shipped_corpus_path()) == ops
    with pytest.raises(corpus.CorpusParseError):
        corpus.from_csv("bad,header\n")
    # the reference's x10 typo on row 25 still passes the gate
    typo = [op if i != 25 else op.__class__(**{**op.__dict__, "flops_published": "3.77487e+09"}) for i, op in enumerate(ops)]
    assert corpus.corpus_gate(typo) == []


def test_recover_pad():
    assert corpus.recover_pad(5, 1, 28, 28) == 2
    assert corpus.recover_pad(11, 4, 227, 55) == 0
    with pytest.raises(corpus.CorpusParseError):
        corpus.recover_pad(3, 1, 5, 4)


def test_ndarray_basics_and_convert_roundtrip():
    a = nda_from_np(NCHW, np.arange(24, dtype=np.float32).reshape(1, 2, 3, 4))
    assert a.at(0, 1, 2, 3) == 23.0
    nhwc = DimsSpec.row_major(("img", "y", "x", "chan"), (1, 3, 4, 8))
    b = convert_format(a, nhwc)
    assert b.dims.sizes == (1, 3, 4, 8) and b.at(0, 2, 3, 1) == 23.0 and b.at(0, 0, 0, 5) == 0.0
    back = convert_format(b, a.dims)
    assert np.array_equal(back.elems, a.elems)
    assert dims_check(a.dims, nhwc) is not None and dims_check(a.dims, a.dims) is None
    assert make_nda(["k"], [3]).to_np().tolist() == [0, 0, 0]


def test_tune_params_string_roundtrip_and_reference_form():
    p = TuneParams(mnt=(2, 2), mnb=(4, 4), kb=1, vw=2, use_local_filts=True, use_local_in=False, bn=96, split_k=4, swap_ab=True)
    s = p.to_string()
    assert s.startswith("MNt=2:2,MNb=4:4,Kb=1,vw=2,lf=1,li=0")
    assert TuneParams.from_string(s) == p
    ref_form = TuneParams.from_string("MNt=8:8,MNb=16:16,Kb=4,vw=4,lf=1,li=1")
    assert ref_form.mnt == (8, 8) and ref_form.bn == 128 and not ref_form.swap_ab
    for bad in ("MNt=2:2", "nonsense"):
        with pytest.raises(CuclgenError):
            TuneParams.from_string(bad)
    with pytest.raises(CuclgenError):
        TuneParams(mnb=(64, 32))
    with pytest.raises(CuclgenError):
        TuneParams(mnt=(4, 2), vw=4)


def test_variant_rank_order_and_heuristic():
    assert [v.name for v in variants_for_kind("Convolution")] == ["conv_fc_stream", "conv_fc", "conv_1x1", "conv_umma",
                                                                  "conv_tiled", "conv_wino", "conv_simple"]
    g = g_of(6, 1, 0, 16, (2, 8, 6, 6))
    assert select_variant(g.node("conv"), g.edges)[0].name == "conv_fc_stream"  # batch <= 8: weight streaming
    g = g_of(6, 1, 0, 16, (20, 8, 6, 6))
    assert select_variant(g.node("conv"), g.edges)[0].name == "conv_fc"
    g = g_of(3, 1, 0, 16, (2, 7, 3, 3))  # ic*h*w = 63: no 16-byte rows
    assert select_variant(g.node("conv"), g.edges)[0].name == "conv_fc"
    g = g_of(1, 1, 0, 16, (2, 8, 6, 6))
    assert select_variant(g.node("conv"), g.edges)[0].name == "conv_1x1"
    g = g_of(3, 1, 1, 16, (1, 4, 8, 8))
    assert select_variant(g.node("conv"), g.edges)[0].name == "conv_umma"


def test_variant_applicability_and_generate():
    g = g_of(3, 1, 1, 2, (1, 1, 5, 5))
    node = g.node("conv")
    assert VARIANTS["conv_tiled"].applies(node, g.edges, DEFAULT_TUNE) is not None  # OC 2 < MNt 4
    with pytest.raises(Inapplicable):
        VARIANTS["conv_tiled"].generate(node, g.edges, DEFAULT_TUNE)
    plan = VARIANTS["conv_simple"].generate(node, g.edges, DEFAULT_TUNE)
    assert plan.name == "conv_simple_b1_ic1_y5_x5_oc2_k3_s1_p1"
    assert VARIANTS["conv_umma"].required_formats(node, g.edges, DEFAULT_TUNE).inputs == {}
    relu = with_fused(g, "conv", "relu").node("conv")
    assert VARIANTS["conv_simple"].generate(relu, g.edges, DEFAULT_TUNE).desc.act == 1
    bad = with_fused(g, "conv", "tanh").node("conv")
    assert VARIANTS["conv_simple"].applies(bad, g.edges, DEFAULT_TUNE) is not None


def test_every_corpus_op_has_candidates():
    for bt in (1, 5, 20):
        for op in corpus.corpus(bt):
            g = with_fused(op.graph(), "conv", "relu")
            cands = tuner.candidates(g.node("conv"), g.edges)
            assert len(cands) >= 3
            names = {v.name for v, _ in cands}
            assert {"conv_simple", "conv_umma"} <= names


def test_op_signature():
    g = g_of(11, 4, 0, 96, (5, 3, 227, 227))
    assert tuner.op_signature(g.node("conv"), g.edges) == "conv:k11:s4:p0:oc96:in5x3x227x227"
    gr = with_fused(g, "conv", "relu")
    assert tuner.op_signature(gr.node("conv"), gr.edges).endswith(":relu")


def test_select_variant_db_record_wins():
    g = g_of(3, 1, 1, 16, (1, 4, 8, 8))
    node = g.node("conv")
    params = TuneParams(mnt=(2, 2), mnb=(8, 8), kb=1, vw=2)
    db = tuner.TuneDB()
    db.add(tuner.TuneRecord(tuner.op_signature(node, g.edges), "conv_tiled", params, 123, CostReport()))
    v, got = select_variant(node, g.edges, db)
    assert v.name == "conv_tiled" and got == params


def test_db_roundtrip_and_errors(tmp_path):
    db = tuner.TuneDB()
    db.add(tuner.TuneRecord("conv:k3:s1:p1:oc16:in1x4x8x8", "conv_umma", TuneParams(bn=64, split_k=2), 1234.5, CostReport()))
    db.add(tuner.TuneRecord("conv:k1:s1:p0:oc8:in1x8x4x4", "conv_tiled", TuneParams((2, 2), (4, 4), 1, 2, True, False), 77, CostReport()))
    path = tmp_path / "tune.db"
    tuner.save_db(db, path)
    text = path.read_text()
    assert text.startswith(tuner.DB_HEADER + "\n") and "MNt=2:2,MNb=4:4,Kb=1,vw=2,lf=1,li=0" in text
    loaded = tuner.load_db(path)
    assert loaded == db
    tuner.save_db(loaded, tmp_path / "tune2.db")
    assert (tmp_path / "tune2.db").read_text() == text
    (tmp_path / "bad.db").write_text("not a tunedb\n")
    with pytest.raises(tuner.FormatVersionMismatch):
        tuner.load_db(tmp_path / "bad.db")
    (tmp_path / "bad.db").write_text(tuner.DB_HEADER + "\nonly\ttwo\n")
    with pytest.raises(tuner.FormatVersionMismatch):
        tuner.load_db(tmp_path / "bad.db")
    with pytest.raises(tuner.IoError):
        tuner.load_db(tmp_path / "missing.db")


def test_db_reads_reference_written_records(tmp_path):
    path = tmp_path / "ref.db"
    path.write_text(tuner.DB_HEADER + "\nconv:k11:s4:p0:oc96:in5x3x227x227\tconv_tiled\tMNt=8:8,MNb=16:16,Kb=4,vw=4,lf=1,li=1\t48211\tmodel\n")
    rec = tuner.load_db(path).records["conv:k11:s4:p0:oc96:in5x3x227x227"]
    assert rec.variant == "conv_tiled" and rec.params.mnt == (8, 8) and rec.cost == 48211


def test_db_concurrent_saves(tmp_path):
    dbs = []
    for i in range(4):
        db = tuner.TuneDB()
        db.add(tuner.TuneRecord(f"sig{i}", "conv_simple", DEFAULT_TUNE, i, CostReport()))
        dbs.append(db)
    ts = [threading.Thread(target=tuner.save_db, args=(db, tmp_path / f"db{i}")) for i, db in enumerate(dbs)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert all(tuner.load_db(tmp_path / f"db{i}") == db for i, db in enumerate(dbs))


def test_model_objective_rejected():
    g = g_of(3, 1, 1, 16, (1, 4, 8, 8))
    with pytest.raises(CuclgenError):
        tuner.sweep(g.node("conv"), g.edges, objective="model")


def test_tolerance_rule():
    assert tuner.tolerance_for(4096).rel_tol == 1e-5 and tuner.tolerance_for(4097).rel_tol == 1e-3


def test_bf16_mode_params_and_applicability():
    """bf16 mode (TuneParams.prec = 1, key ``pr``): TMA tcgen05 kernel with pixels on M only."""
    p = TuneParams.from_string("MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,BN=64,sk=1,sw=0,dr=0,tm=1,pr=1")
    assert p.prec == 1 and p.to_string().endswith(",pr=1") and TuneParams.from_string(p.to_string()) == p
    assert TuneParams().to_string().count("pr=") == 0
    g = g_of(3, 1, 1, 64, (2, 32, 13, 13))
    node = g.node("conv")
    assert VARIANTS["conv_umma"].applies(node, g.edges, p) is None
    assert VARIANTS["conv_umma"].generate(node, g.edges, p).desc.prec == 1
    for bad in (TuneParams(bn=64, prec=1), TuneParams(bn=64, tma=1, swap_ab=True, prec=1),
                TuneParams(bn=96, tma=1, prec=1), TuneParams(bn=64, tma=1, occ=2, prec=1)):
        assert VARIANTS["conv_umma"].applies(node, g.edges, bad) is not None, bad
    assert VARIANTS["conv_simple"].applies(node, g.edges, TuneParams(prec=1)) is not None
    cands = tuner.candidates(node, g.edges, prec=1)
    assert cands and all(p.prec == 1 and v.name in ("conv_umma", "conv_1x1") for v, p in cands)
    assert tuner.tolerance_for(9999, prec=1).rel_tol == 4e-3 and tuner.tolerance_for(100).rel_tol == 1e-5


def test_direct_nchw_operand_paths_applicability():
    """tm=3 (1x1 straight from NCHW) and tm=4 (k x k stride 1 straight from NCHW): TMA needs
    16-byte global strides, so h*w*4 (tm=3) / w*4 (tm=4) must be multiples of 16."""
    one = g_of(1, 1, 0, 64, (2, 96, 28, 28))       # h*w = 784: ok
    odd = g_of(1, 1, 0, 64, (2, 96, 13, 13))       # 169: no
    k3 = g_of(3, 1, 1, 64, (2, 64, 28, 28))        # w = 28: ok
    k3odd = g_of(3, 1, 1, 64, (2, 64, 27, 27))     # w = 27: no
    k3s2 = g_of(3, 2, 1, 64, (2, 64, 28, 28))      # stride 2: no
    ok = lambda g, p: VARIANTS["conv_umma"].applies(g.node("conv"), g.edges, p) is None  # noqa: E731
    assert ok(one, TuneParams(bn=64, tma=3)) and not ok(odd, TuneParams(bn=64, tma=3))
    assert not ok(k3, TuneParams(bn=64, tma=3))    # tm=3 is 1x1 only
    assert ok(k3, TuneParams(bn=64, tma=4)) and not ok(k3odd, TuneParams(bn=64, tma=4))
    assert not ok(k3s2, TuneParams(bn=64, tma=4)) and not ok(one, TuneParams(bn=64, tma=4))
    assert not ok(k3, TuneParams(bn=64, tma=4, swap_ab=True))
    assert ok(k3, TuneParams(bn=64, tma=4, prec=1)) and ok(one, TuneParams(bn=64, tma=3, prec=1))
    n_tm34 = sum(1 for v, p in tuner.candidates(k3.node("conv"), k3.edges) if p.tma == 4)
    assert n_tm34 > 0
