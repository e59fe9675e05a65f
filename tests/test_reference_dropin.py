"""The drop-in, proven on the real reference: the UNMODIFIED reference package
(cuclgen 0.1.0, installed into baseline/_ref by baseline/fetch_ref.sh) with the
reference-side binding integration/cuclgen_b200.py applied, driven through
the reference's OWN entry points:

* tests/helpers.run_conv_variant (pkg/tests/helpers.py:59-79): build graph ->
  cuclgen.runner.execute_node -> cuclgen.oracle.ref_conv -> compare, for the
  reference's own variants (conv_simple / conv_tiled with random tile params /
  conv_1x1 / conv_fc) on the reference's own random cases (random_conv_case);
* cuclgen.runner.validate_node (runner.py:109-115) on corpus ops;
* cuclgen.tuner.load_db on the shipped B200 TuneDB (tuner.py:280 rejects
  unknown variants: the binding registers conv_umma / conv_fc_stream) and
  cuclgen.variants.select_variant -> execute_node at FULL size on the tuned
  B200 tile, checked by the reference's compare at its tolerance.

The CPU tests check the binding loads, registers and parses without a GPU.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SITE = os.path.join(ROOT, "baseline", "_ref", "site")
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "tests")
FP32_DB = os.path.join(ROOT, "paper_1611_06945_b200", "data", "tunedb_b200_fp32.tsv")


def _reference():
    if not os.path.isdir(os.path.join(REF_SITE, "cuclgen")):
        pytest.fail("baseline/_ref is not installed: run baseline/fetch_ref.sh in the build container")
    for p in (REF_SITE, REF_TESTS, ROOT):
        if p not in sys.path:
            sys.path.insert(0, p)
    import cuclgen
    import cuclgen.corpus
    import cuclgen.frontend
    import cuclgen.oracle
    import cuclgen.runner
    import cuclgen.tuner
    import cuclgen.variants  # noqa: F401

    from integration import cuclgen_b200

    cuclgen_b200.install(cuclgen)
    import helpers  # the reference's tests/helpers.py: imported after install, so it binds the patched execute_node

    return cuclgen, helpers


def test_binding_installs_and_reads_b200_db_on_cpu():
    cuclgen, _ = _reference()
    import cuclgen.tuner as T
    import cuclgen.variants as V

    assert "conv_umma" in V.VARIANTS and "conv_fc_stream" in V.VARIANTS
    db = T.load_db(FP32_DB)
    assert len(db.records) >= 129
    rec = db.records["conv:k5:s1:p2:oc256:in20x96x27x27:relu"]
    assert rec.variant in V.VARIANTS and ",BN=" in rec.params.to_string()  # tuned tile kept verbatim
    assert V.TuneParams.from_string(rec.params.to_string()) == rec.params
    assert type(V.TuneParams.from_string("MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1")) is V.TuneParams
    # the reference's heuristic (no DB) is unchanged: most specialized reference variant first
    from dataclasses import replace

    g = replace(cuclgen.corpus.corpus()[42], batch=20).graph()
    g.nodes = [replace(n, fused_activation="relu") if n.name == "conv" else n for n in g.nodes]
    assert V.select_variant(g.node("conv"), g.edges)[0].name == "conv_tiled"
    v, p = V.select_variant(g.node("conv"), g.edges, db)
    assert v.name in ("conv_umma", "conv_1x1") and getattr(p, "bn", None)


@pytest.mark.gpu
def test_reference_helpers_run_conv_variant_on_b200(cuda):
    """The reference's own test helper + random cases, every reference variant, on the B200."""
    cuclgen, helpers = _reference()
    rng = np.random.default_rng(2024)
    ran = {}
    for _ in range(25):
        p, in_dims = helpers.random_conv_case(rng)
        for vname in ("conv_simple", "conv_tiled", "conv_1x1", "conv_fc"):
            params = helpers.random_tile_params(rng) if vname == "conv_tiled" else cuclgen.variants.DEFAULT_TUNE
            for fused in (None, "relu"):
                try:
                    r = helpers.run_conv_variant(p, in_dims, vname, params, fused=fused)
                except cuclgen.variants.Inapplicable:
                    continue  # the reference applies() but the B200 kernel does not (e.g. an oversize tile)
                if r is None:
                    continue
                res, got, ref, report = r
                assert res.ok, (vname, p, in_dims, params.to_string(), res)
                assert report.wall_ns > 0
                ran[vname] = ran.get(vname, 0) + 1
    assert ran.get("conv_simple", 0) >= 40 and ran.get("conv_tiled", 0) >= 20
    assert ran.get("conv_1x1", 0) >= 2 and ran.get("conv_fc", 0) >= 1, ran


@pytest.mark.gpu
def test_reference_validate_node_on_downscaled_corpus(cuda):
    cuclgen, _ = _reference()
    import cuclgen.runner as R
    import cuclgen.tuner as T
    import cuclgen.variants as V

    for i, op in enumerate(cuclgen.corpus.corpus()):
        g = cuclgen.frontend.conv_graph(*T.downscale_conv(op.conv_params, op.input_dims))  # the tuner's twin
        node = g.node("conv")
        v, p = V.select_variant(node, g.edges)
        res, report = R.validate_node(node, g.edges, v, p)
        assert res.ok, (i, v.name, res)


@pytest.mark.gpu
@pytest.mark.parametrize("row,batch", [(34, 1), (42, 5), (38, 20), (4, 20), (25, 1), (13, 20), (41, 1)])
def test_reference_execute_node_full_size_on_tuned_b200_tile(cuda, row, batch):
    """select_variant over the shipped B200 DB (loaded by the reference's load_db) ->
    the reference's execute_node (patched) at full size -> the reference's
    node_reference + compare at the reference tolerance."""
    from dataclasses import replace

    cuclgen, _ = _reference()
    import cuclgen.oracle as O
    import cuclgen.runner as R
    import cuclgen.tuner as T
    import cuclgen.variants as V

    db = T.load_db(FP32_DB)
    op = replace(cuclgen.corpus.corpus()[row], batch=batch)
    g = op.graph()
    g.nodes = [replace(n, fused_activation="relu") if n.name == "conv" else n for n in g.nodes]
    node = g.node("conv")
    sig = T.op_signature(node, g.edges)
    assert sig in db.records
    v, p = V.select_variant(node, g.edges, db)
    inputs = R.node_test_inputs(node, g.edges, f"bench:{sig}")
    got, report = R.execute_node(node, g.edges, inputs, v, p)
    want = R.node_reference(node, g.edges, inputs)
    res = O.compare(got, want, O.tolerance_for(R.conv_reduction_terms(node, g.edges)))
    assert res.ok, (sig, v.name, p.to_string(), res)
