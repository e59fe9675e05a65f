"""Golden vectors for the whole-network path, made by running the REFERENCE.

Run in the build container (the reference is not shipped to the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_net_golden.py

Records (tests/golden/net_cases.json + net_cases.npz):
* ``nets``: for each network file under paper_1611_06945_b200/data/nets, the
  reference's parse_net result (nodes, edge shapes), schedule order,
  fuse_activations result and pretty_print text (cuclgen/frontend.py:334-434,
  graphopt.py:39-86);
* ``pool``: reference ref_pool_max (oracle.py:100-116) outputs on seeded noise;
* ``relu``: reference ref_relu (oracle.py:119-121) on signed data
  (2*noise - 1.1, so about half the inputs clip);
* ``xpose``: reference convert_format (ndarray.py:232-253) for permutations,
  zero-pad growth and crops;
* ``tiny``: the reference's whole-graph run_graph (runner.py:200-249, on its
  SIMT interpreter, check=True) of a small conv/relu/pool network: the sink
  arrays, so the B200 run_graph can be compared to the reference end to end.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from cuclgen import graphopt as rgraphopt
from cuclgen import oracle as roracle
from cuclgen import runner as rrunner
from cuclgen.frontend import PoolParams, parse_net, pretty_print
from cuclgen.ndarray import DimsSpec, convert_format, nda_from_np

HERE = os.path.dirname(os.path.abspath(__file__))
NETS = os.path.join(HERE, "..", "..", "paper_1611_06945_b200", "data", "nets")

TINY_NET = """
input: "data"
input_dim: 2
input_dim: 3
input_dim: 12
input_dim: 12
layer { name: "conv1" type: "Convolution" bottom: "data" top: "c1"
  convolution_param { num_output: 8 kernel_size: 3 pad: 1 } }
layer { name: "relu1" type: "ReLU" bottom: "c1" top: "r1" }
layer { name: "pool1" type: "Pooling" bottom: "r1" top: "p1"
  pooling_param { pool: MAX kernel_size: 3 stride: 2 pad: 1 } }
layer { name: "conv2" type: "Convolution" bottom: "p1" top: "c2"
  convolution_param { num_output: 6 kernel_size: 1 } }
layer { name: "relu2" type: "ReLU" bottom: "c2" top: "r2" }
layer { name: "pool2" type: "Pooling" bottom: "r2" top: "p2"
  pooling_param { pool: MAX kernel_size: 2 stride: 2 } }
"""


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()[:16]


def node_rec(n):
    p = n.params
    params = None if p is None else {k: getattr(p, k) for k in ("ksz", "stride", "pad", "out_chans", "func") if hasattr(p, k)}
    return {"name": n.name, "kind": n.kind, "params": params, "inputs": list(n.inputs), "outputs": list(n.outputs),
            "fused_activation": n.fused_activation}


def main():
    manifest = {"nets": {}, "pool": [], "relu": [], "xpose": [], "tiny": {}}
    arrays = {}
    for fn in sorted(os.listdir(NETS)):
        text = open(os.path.join(NETS, fn)).read()
        g = parse_net(text)
        fused = rgraphopt.fuse_activations(g)
        manifest["nets"][fn] = {
            "nodes": [node_rec(n) for n in g.nodes],
            "edges": {e: [list(s.names), list(s.sizes)] for e, s in g.edges.items()},
            "sources": list(g.sources),
            "sinks": list(g.sinks),
            "schedule": rgraphopt.schedule(g),
            "fused_nodes": [node_rec(n) for n in fused.nodes],
            "fused_schedule": rgraphopt.schedule(fused),
            "pretty": pretty_print(g),
        }
    # pooling
    pool_cases = [(2, 3, 13, 13, 3, 2, 0), (1, 4, 12, 12, 3, 2, 1), (2, 5, 9, 7, 2, 2, 0), (1, 2, 6, 6, 6, 1, 0),
                  (1, 3, 8, 8, 3, 1, 1), (3, 2, 11, 10, 4, 3, 2), (1, 1, 5, 5, 5, 5, 4)]
    for i, (b, c, h, w, k, s, p) in enumerate(pool_cases):
        seed = f"pool{i}"
        x = roracle.noise(("img", "chan", "y", "x"), (b, c, h, w), roracle.seed_for(seed))
        y = roracle.ref_pool_max(x, PoolParams(ksz=k, stride=s, pad=p))
        key = f"pool{i}"
        arrays[key] = y.to_np()
        manifest["pool"].append({"id": key, "seed": seed, "dims": [b, c, h, w], "ksz": k, "stride": s, "pad": p,
                                 "in_digest": digest(x.to_np()), "out_shape": list(y.to_np().shape)})
    # relu on signed data
    for i, shape in enumerate([(2, 3, 5, 7), (1, 16, 4, 4), (3, 1, 1, 5)]):
        seed = f"relu{i}"
        x = roracle.noise(("img", "chan", "y", "x"), shape, roracle.seed_for(seed))
        xs = (x.to_np() * np.float32(2.0) - np.float32(1.1)).astype(np.float32)
        y = roracle.ref_relu(nda_from_np(("img", "chan", "y", "x"), xs))
        key = f"relu{i}"
        arrays[key] = y.to_np()
        manifest["relu"].append({"id": key, "seed": seed, "shape": list(shape), "in_digest": digest(xs)})
    # layout conversion
    xcases = [
        (("img", "chan", "y", "x"), (2, 5, 4, 3), ("img", "y", "x", "chan"), (2, 4, 3, 5)),       # NCHW -> NHWC
        (("img", "chan", "y", "x"), (2, 5, 4, 3), ("img", "y", "x", "chan"), (2, 4, 3, 8)),       # + pad chan
        (("img", "chan", "y", "x"), (1, 3, 6, 6), ("img", "chan", "y", "x"), (1, 4, 5, 8)),       # grow + crop
        (("out_chan", "in_chan", "y", "x"), (7, 3, 3, 3), ("in_chan", "y", "x", "out_chan"), (3, 3, 3, 8)),  # k-major filts
        (("a", "b"), (37, 45), ("b", "a"), (45, 37)),                                               # 2-D transpose
        (("a", "b", "c"), (3, 40, 33), ("c", "a", "b"), (33, 3, 40)),                               # 3-D rotate
        (("img", "y", "x", "chan"), (2, 4, 3, 8), ("img", "chan", "y", "x"), (2, 5, 4, 3)),       # NHWC -> NCHW + crop
    ]
    for i, (sn, ss, dn, ds) in enumerate(xcases):
        seed = f"xpose{i}"
        x = roracle.noise(sn, ss, roracle.seed_for(seed))
        y = convert_format(x, DimsSpec.row_major(dn, ds))
        key = f"xpose{i}"
        arrays[key] = y.to_np()
        manifest["xpose"].append({"id": key, "seed": seed, "src": [list(sn), list(ss)], "dst": [list(dn), list(ds)],
                                  "in_digest": digest(x.to_np())})
    # tiny whole graph through the reference's own run_graph
    g = parse_net(TINY_NET)
    res = rrunner.run_graph(g, seed="tiny", check=True, keep_sinks=True)
    assert res.all_checks_pass
    manifest["tiny"] = {"net": TINY_NET, "seed": "tiny", "sinks": {}, "order": None}
    plan = rrunner.plan_graph(g)
    manifest["tiny"]["order"] = plan.order
    manifest["tiny"]["choices"] = {k: [v, p.to_string()] for k, (v, p) in plan.choices.items()}
    for e, nda in res.sink_buffers.items():
        arrays[f"tiny_{e}"] = nda.to_np()
        manifest["tiny"]["sinks"][e] = {"checksum": res.checksums[e], "shape": list(nda.to_np().shape)}
    with open(os.path.join(HERE, "net_cases.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "net_cases.npz"), **arrays)
    print(f"{len(manifest['nets'])} nets, {len(pool_cases)} pool, {len(manifest['relu'])} relu, "
          f"{len(xcases)} xpose, tiny sinks {list(manifest['tiny']['sinks'])}")


if __name__ == "__main__":
    main()
