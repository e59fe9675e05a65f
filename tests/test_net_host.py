"""Whole-network path, host side (no GPU): the network parser, graph rewrites,
schedule and planning mirror the reference (pinned by tests/golden/net_cases.*,
made by importing cuclgen), and the CPU oracle for pool / ReLU / conversion
matches the reference's outputs bit-exactly.  Restates the reference's own
tests where they apply: pkg/tests/test_frontend.py:36-99, test_graphopt.py."""

import json
import os

import numpy as np
import pytest

from oracle import conv_ref, net_ref
from paper_1611_06945_b200 import backend, graphopt, runner
from paper_1611_06945_b200.frontend import (KIND_ACT, KIND_CONVERT, ActParams, ComputeGraph, ConvertParams,
                                            DanglingBottom, NetSyntaxError, OpNode, UnknownLayerType, parse_net,
                                            pretty_print)
from paper_1611_06945_b200.ndarray import DimsSpec

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "net_cases.json")))
ARR = np.load(os.path.join(HERE, "golden", "net_cases.npz"))
NETS = os.path.join(os.path.dirname(HERE), "paper_1611_06945_b200", "data", "nets")
HDR = 'input: "d"\ninput_dim: 1\ninput_dim: 1\ninput_dim: 4\ninput_dim: 4\n'


def _node_rec(n):
    p = n.params
    params = None if p is None else {k: getattr(p, k) for k in ("ksz", "stride", "pad", "out_chans", "func") if hasattr(p, k)}
    return {"name": n.name, "kind": n.kind, "params": params, "inputs": list(n.inputs), "outputs": list(n.outputs),
            "fused_activation": n.fused_activation}


@pytest.mark.parametrize("fn", sorted(GOLD["nets"]))
def test_network_files_parse_like_the_reference(fn):
    want = GOLD["nets"][fn]
    g = parse_net(open(os.path.join(NETS, fn)).read())
    assert [_node_rec(n) for n in g.nodes] == want["nodes"]
    assert {e: [list(s.names), list(s.sizes)] for e, s in g.edges.items()} == want["edges"]
    assert g.sources == want["sources"] and g.sinks == want["sinks"]
    assert graphopt.schedule(g) == want["schedule"]
    fused = graphopt.fuse_activations(g)
    assert [_node_rec(n) for n in fused.nodes] == want["fused_nodes"]
    assert graphopt.schedule(fused) == want["fused_schedule"]
    assert pretty_print(g) == want["pretty"]


@pytest.mark.parametrize("fn", sorted(GOLD["nets"]))
def test_pretty_print_roundtrip(fn):
    g1 = parse_net(open(os.path.join(NETS, fn)).read())
    text = pretty_print(g1)
    g2 = parse_net(text)
    assert pretty_print(g2) == text and g2.edges == g1.edges
    assert [n.params for n in g2.nodes] == [n.params for n in g1.nodes]


def test_parse_errors():
    with pytest.raises(NetSyntaxError):
        parse_net('input: "d"\ninput_dim: 1\ninput_dim: 1\ninput_dim: 1')
    with pytest.raises(UnknownLayerType):
        parse_net(HDR + 'layer { name: "s" type: "Softmax" bottom: "d" top: "o" }')
    with pytest.raises(DanglingBottom):
        parse_net(HDR + 'layer { name: "r" type: "ReLU" bottom: "nope" top: "o" }')
    with pytest.raises(NetSyntaxError):
        parse_net('layer { name: "c" type: "Convolution" bottom: "d" top: "o" blobs_lr: 1 }')
    with pytest.raises(NetSyntaxError):
        parse_net(HDR + 'layer { name: "r" type: "ReLU" bottom: "d" top: "d" }')
    with pytest.raises(NetSyntaxError):
        parse_net(HDR + 'layer { name: "p" type: "Pooling" bottom: "d" top: "o" pooling_param { pool: AVE kernel_size: 2 } }')
    with pytest.raises(NetSyntaxError):
        parse_net(HDR + 'layer { name: "c" type: "Convolution" bottom: "d" top: "o" convolution_param { kernel_size: 3 } }')
    with pytest.raises(NetSyntaxError):
        parse_net('input: "d\ninput_dim: 1')


def test_input_only_and_comments():
    g = parse_net('# just an input\ninput: "data"\ninput_dim: 1\ninput_dim: 2\ninput_dim: 3\ninput_dim: 4  # trailing')
    assert len(g.nodes) == 1 and g.sinks == g.sources == ["data"]


def _synth(edges, nodes):
    g = ComputeGraph()
    for e in edges:
        g.edges[e] = DimsSpec.row_major(["k"], [4])
    for name, ins, outs in nodes:
        g.nodes.append(OpNode(name, KIND_ACT, ActParams(), tuple(ins), tuple(outs)))
    g.recompute_endpoints()
    return g


def test_schedule_chain_diamond_cycle_and_declaration_ties():
    g = _synth(["e0", "e1", "e2", "e3"], [("a", ["e0"], ["e1"]), ("b", ["e1"], ["e2"]), ("c", ["e2"], ["e3"])])
    assert graphopt.schedule(g) == ["a", "b", "c"]
    g = _synth(["s", "ab", "ac", "bd", "cd", "o"],
               [("a", ["s"], ["ab", "ac"]), ("b", ["ab"], ["bd"]), ("c", ["ac"], ["cd"]), ("d", ["bd", "cd"], ["o"])])
    assert graphopt.schedule(g) == ["a", "b", "c", "d"]
    g = _synth(["e0", "e1", "e2", "e3"], [("b", ["e1"], ["e2"]), ("a", ["e0"], ["e1"]), ("x", ["e0"], ["e3"])])
    assert graphopt.schedule(g) == ["a", "x", "b"]
    g = _synth(["x", "y"], [("a", ["x"], ["y"]), ("b", ["y"], ["x"])])
    with pytest.raises(graphopt.CycleDetected):
        graphopt.schedule(g)


NET = 'input: "d"\ninput_dim: 1\ninput_dim: 3\ninput_dim: 8\ninput_dim: 8\n' + (
    'layer { name: "conv1" type: "Convolution" bottom: "d" top: "c1" convolution_param { num_output: 4 kernel_size: 3 pad: 1 } }\n'
    'layer { name: "relu1" type: "ReLU" bottom: "c1" top: "r1" }\n'
    'layer { name: "pool1" type: "Pooling" bottom: "r1" top: "p1" pooling_param { pool: MAX kernel_size: 2 stride: 2 } }\n')


def test_fuse_rules():
    g = parse_net(NET)
    f = graphopt.fuse_activations(g)
    assert [n.name for n in f.nodes] == ["d_input", "conv1", "pool1"]
    assert f.node("conv1").fused_activation == "relu" and f.node("conv1").outputs == ("r1",) and "c1" not in f.edges
    g2 = parse_net(NET + 'layer { name: "conv2" type: "Convolution" bottom: "c1" top: "c2" convolution_param { num_output: 2 kernel_size: 1 } }\n')
    assert graphopt.fuse_activations(g2).node("conv1").fused_activation is None
    g3 = parse_net(NET)
    g3.sinks = ["c1", "p1"]
    assert graphopt.fuse_activations(g3).node("conv1").fused_activation is None


def test_insert_conversions_and_alloc():
    g = parse_net(NET)
    want_in = DimsSpec.row_major(("img", "y", "x", "chan"), (1, 8, 8, 4))
    want_out = DimsSpec.row_major(("img", "y", "x", "chan"), (1, 8, 8, 8))
    g2 = graphopt.insert_conversions(g, {"conv1": graphopt.VariantFormats({"d": want_in}, want_out)})
    names = [n.name for n in g2.nodes]
    assert names == ["d_input", "conv1__cv_in0", "conv1", "conv1__cv_out", "relu1", "pool1"]
    assert g2.node("conv1").inputs[0] == "d__for_conv1" and g2.node("conv1").outputs == ("c1__raw",)
    assert g2.edges["c1__raw"] == want_out and g2.node("conv1__cv_out").params == ConvertParams(g.edges["c1"])
    with pytest.raises(graphopt.IncompatibleFormats):
        graphopt.insert_conversions(g, {"conv1": graphopt.VariantFormats({"d": DimsSpec.row_major(("a", "b"), (1, 2))})})
    ap = graphopt.alloc_plan(g2)
    assert len(ap.entries) == len(g2.edges) and ap.total_elems == sum(s.num_elems for s in g2.edges.values())


@pytest.mark.parametrize("fn", sorted(GOLD["nets"]))
def test_plan_graph_networks(fn):
    g = parse_net(open(os.path.join(NETS, fn)).read())
    plan = runner.plan_graph(g)
    want = [n for n in GOLD["nets"][fn]["fused_schedule"] if not n.endswith("_input")]
    assert plan.order == want  # canonical-format variants: no conversion nodes
    for name in plan.order:
        kind = plan.graph.node(name).kind
        v = plan.choices[name][0]
        assert (kind, v) in {("Convolution", "conv_fc"), ("Convolution", "conv_fc_stream"), ("Convolution", "conv_1x1"), ("Convolution", "conv_umma"),
                             ("Pooling", "pool_max"), ("Activation", "activation")}


def test_plan_graph_with_conversion_uses_xpose():
    g = parse_net(NET)
    cv = OpNode("cv", KIND_CONVERT, ConvertParams(DimsSpec.row_major(("img", "y", "x", "chan"), (1, 4, 4, 4))), ("p1",), ("p1t",))
    g.nodes.append(cv)
    g.edges["p1t"] = None
    g.recompute_endpoints()
    from paper_1611_06945_b200.frontend import infer_shapes

    g = infer_shapes(g, g.edges["d"])
    plan = runner.plan_graph(g)
    assert plan.choices["cv"][0] == "xpose"
    d = plan.insts["cv"].desc
    assert d.ndim == 4 and list(d.out_sizes)[:4] == [1, 4, 4, 4] and list(d.src_strides)[:4] == [64, 4, 1, 16]


def test_xpose_desc_rejects_mismatched_names():
    with pytest.raises(Exception):
        backend.xpose_desc(("a", "b"), (2, 3), (3, 1), ("a", "c"), (2, 3))


# -------------------------------------------------------------------- oracle pinned to the reference

@pytest.mark.parametrize("case", GOLD["pool"], ids=[c["id"] for c in GOLD["pool"]])
def test_oracle_pool_matches_reference(case):
    x = conv_ref.noise(tuple(case["dims"]), conv_ref.seed_for(case["seed"]))
    got = net_ref.ref_pool_max(x, case["ksz"], case["stride"], case["pad"])
    assert np.array_equal(got, ARR[case["id"]])


@pytest.mark.parametrize("case", GOLD["relu"], ids=[c["id"] for c in GOLD["relu"]])
def test_oracle_relu_matches_reference(case):
    x = conv_ref.noise(tuple(case["shape"]), conv_ref.seed_for(case["seed"])) * np.float32(2.0) - np.float32(1.1)
    got = net_ref.ref_relu(x.astype(np.float32))
    assert np.array_equal(got, ARR[case["id"]]) and (got == 0).any() and (got > 0).any()


@pytest.mark.parametrize("case", GOLD["xpose"], ids=[c["id"] for c in GOLD["xpose"]])
def test_oracle_convert_matches_reference(case):
    (sn, ss), (dn, ds) = case["src"], case["dst"]
    x = conv_ref.noise(tuple(ss), conv_ref.seed_for(case["seed"]))
    got = net_ref.convert_format(x, sn, dn, ds)
    assert np.array_equal(got, ARR[case["id"]])
