"""Whole-network path on the B200: the pool / ReLU / conversion kernels through
the C ABI against the reference's golden outputs (bit-exact: they are exact
ops) and the CPU oracle on larger shapes, and run_graph end to end — the
reference's own run_graph output for a tiny network, and every node of
AlexNet / NiN / GoogLeNet-3a checked against the oracle at the reference
tolerance (rel 1e-5 for ic*k*k <= 4096 else 1e-3, cuclgen/oracle.py:31-38)."""

import json
import os

import numpy as np
import pytest

from oracle import conv_ref, net_ref

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "net_cases.json")))
ARR = np.load(os.path.join(HERE, "golden", "net_cases.npz"))
NETS = os.path.join(os.path.dirname(HERE), "paper_1611_06945_b200", "data", "nets")


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _pool(x, k, s, p):
    import torch

    from paper_1611_06945_b200 import backend

    b, c, h, w = x.shape
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    y = torch.full((b, c, oh, ow), float("nan"), device="cuda")
    backend.pool_max_fwd(backend.PoolDesc(b, c, h, w, k, s, p, oh, ow), _dev(x), y)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def _xpose(x, sn, dn, ds):
    import torch

    from paper_1611_06945_b200 import backend

    strides = [int(np.prod(x.shape[i + 1:])) for i in range(x.ndim)]
    y = torch.full(tuple(ds), float("nan"), device="cuda")
    backend.xpose(backend.xpose_desc(sn, x.shape, strides, dn, ds), _dev(x), y)
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("case", GOLD["pool"], ids=[c["id"] for c in GOLD["pool"]])
def test_pool_matches_reference(cuda, case):
    x = conv_ref.noise(tuple(case["dims"]), conv_ref.seed_for(case["seed"]))
    assert np.array_equal(_pool(x, case["ksz"], case["stride"], case["pad"]), ARR[case["id"]])


@pytest.mark.parametrize("shape,k,s,p", [((20, 96, 55, 55), 3, 2, 0), ((5, 64, 112, 112), 3, 2, 1),
                                         ((3, 192, 28, 28), 3, 1, 1), ((2, 1000, 6, 6), 6, 1, 0)])
def test_pool_signed_large(cuda, shape, k, s, p):
    x = conv_ref.noise(shape, conv_ref.seed_for(f"pool{shape}"), -1.0, 1.0)
    assert np.array_equal(_pool(x, k, s, p), net_ref.ref_pool_max(x, k, s, p))


@pytest.mark.parametrize("case", GOLD["relu"], ids=[c["id"] for c in GOLD["relu"]])
def test_relu_matches_reference(cuda, case):
    import torch

    from paper_1611_06945_b200 import backend

    x = (conv_ref.noise(tuple(case["shape"]), conv_ref.seed_for(case["seed"])) * np.float32(2.0) - np.float32(1.1)).astype(np.float32)
    xd = _dev(x)
    y = torch.empty_like(xd)
    backend.relu_fwd(xd, y)
    backend.relu_fwd(xd, xd)  # in place
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), ARR[case["id"]]) and np.array_equal(xd.cpu().numpy(), ARR[case["id"]])


def test_relu_vector_and_tail(cuda):
    import torch

    from paper_1611_06945_b200 import backend

    for n in (1, 3, 4, 1027, 1 << 20):
        x = conv_ref.noise((n,), n, -1.0, 1.0)
        xd = _dev(x)
        y = torch.empty_like(xd)
        backend.relu_fwd(xd, y)
        z = torch.empty(n + 1, device="cuda")[1:]  # misaligned: scalar path
        backend.relu_fwd(xd, z)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), net_ref.ref_relu(x)) and np.array_equal(z.cpu().numpy(), net_ref.ref_relu(x))


@pytest.mark.parametrize("case", GOLD["xpose"], ids=[c["id"] for c in GOLD["xpose"]])
def test_xpose_matches_reference(cuda, case):
    (sn, ss), (dn, ds) = case["src"], case["dst"]
    x = conv_ref.noise(tuple(ss), conv_ref.seed_for(case["seed"]))
    assert np.array_equal(_xpose(x, sn, dn, ds), ARR[case["id"]])


@pytest.mark.parametrize("sn,ss,dn,ds", [
    (("img", "chan", "y", "x"), (20, 96, 27, 27), ("img", "y", "x", "chan"), (20, 27, 27, 96)),
    (("img", "y", "x", "chan"), (5, 13, 13, 384), ("img", "chan", "y", "x"), (5, 384, 13, 13)),
    (("out_chan", "in_chan", "y", "x"), (256, 96, 5, 5), ("in_chan", "y", "x", "out_chan"), (96, 5, 5, 256)),
    (("a", "b"), (1000, 4096), ("b", "a"), (4096, 1024)),
    (("img", "chan", "y", "x"), (2, 3, 227, 227), ("img", "y", "x", "chan"), (2, 227, 227, 4)),
    (("a", "b", "c", "d", "e"), (2, 3, 4, 5, 6), ("e", "c", "a", "d", "b"), (7, 4, 2, 5, 3)),
])
def test_xpose_large_and_tiled(cuda, sn, ss, dn, ds):
    x = conv_ref.noise(ss, conv_ref.seed_for(f"x{ss}"), -1.0, 1.0)
    assert np.array_equal(_xpose(x, sn, dn, ds), net_ref.convert_format(x, sn, dn, ds))


def test_tiny_net_matches_reference_run_graph(cuda):
    from paper_1611_06945_b200 import runner
    from paper_1611_06945_b200.frontend import parse_net

    t = GOLD["tiny"]
    res = runner.run_graph(parse_net(t["net"]), seed=t["seed"], check=net_ref.check_node, keep_sinks=True)
    assert all(r.ok for r in res.oracle_checks.values()), res.oracle_checks
    for e, meta in t["sinks"].items():
        got = res.sink_buffers[e].to_np()
        r = conv_ref.compare(got, ARR[f"tiny_{e}"], conv_ref.Tol(2e-5))
        assert r.ok, (e, r)


@pytest.mark.parametrize("fn,batch", [("alexnet.net", 1), ("alexnet.net", 5), ("nin.net", 1), ("googlenet_3a.net", 2)])
def test_network_every_node_vs_oracle(cuda, fn, batch):
    from paper_1611_06945_b200 import runner
    from paper_1611_06945_b200.frontend import infer_shapes, parse_net
    from paper_1611_06945_b200.ndarray import DimsSpec

    g = parse_net(open(os.path.join(NETS, fn)).read())
    d = g.edges["data"]
    g = infer_shapes(g, DimsSpec.row_major(d.names, (batch,) + d.sizes[1:]))
    res = runner.run_graph(g, seed=f"net:{fn}", check=net_ref.check_node)
    bad = {k: v for k, v in res.oracle_checks.items() if not v.ok}
    assert not bad, bad
    assert len(res.oracle_checks) == len(res.node_runs) and all(r.report.wall_ns > 0 for r in res.node_runs)


def test_graph_exec_replay_is_deterministic(cuda):
    import torch

    from paper_1611_06945_b200 import runner
    from paper_1611_06945_b200.frontend import parse_net

    g = parse_net(open(os.path.join(NETS, "googlenet_3a.net")).read())
    ex = runner.GraphExec(runner.plan_graph(g), seed="replay")
    ex.launch()
    torch.cuda.synchronize()
    first = {e: ex.buffers[e].clone() for e in ex.plan.graph.sinks}
    st = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        with torch.cuda.graph(graph, stream=st):
            ex.launch(st.cuda_stream)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    for e, t in first.items():
        assert torch.equal(t, ex.buffers[e]), e


def test_network_bf16_mode_via_bf16_tunedb(cuda):
    """The bf16 TuneDB's records carry pr=1, so plan_graph with it runs every conv node in the
    bf16 mode; each node is checked at the bf16 tolerance (rel 4e-3), pool exactly."""
    from paper_1611_06945_b200 import runner, tuner
    from paper_1611_06945_b200.frontend import parse_net

    db = tuner.load_db(tuner.shipped_db_path("bf16"))
    g = parse_net(open(os.path.join(NETS, "alexnet.net")).read())
    plan = runner.plan_graph(g, db=db)
    assert any(p.prec == 1 for v, p in plan.choices.values() if v.startswith("conv_"))

    def check(node, edges, inputs, got):
        ins = {e: a.to_np() for e, a in inputs.items()}
        want = net_ref.node_reference(node, edges, ins)
        tol = conv_ref.Tol(4e-3) if node.kind == "Convolution" else conv_ref.Tol(0.0, 0.0)
        return conv_ref.compare(got.to_np(), want, tol)

    res = runner.run_graph(g, seed="bf16net", db=db, check=check)
    bad = {k: v for k, v in res.oracle_checks.items() if not v.ok}
    assert not bad, bad
