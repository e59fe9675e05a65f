"""Every candidate the on-device tuner may pick, checked against the float64 oracle.

The tuner (tuner.sweep) validates each candidate against the exact-order
``conv_simple`` kernel on the device before timing it; this test closes the
remaining gap by running the WHOLE candidate list of representative ops --
every variant x tile x split-K / stream-K x operand path x CTA pairs / split-K
clusters / Winograd / space-to-depth the tuner enumerates -- against the CPU
oracle (oracle/conv_ref.py, the reference's ref_conv) at the reference
tolerance (rel 1e-5 up to 4096 reduction terms, cuclgen/oracle.py:31-38), on
signed inputs with a cancellation-aware bound and exact ReLU clipping as well.
The ops are small batches of corpus shapes, so the ~100-300 candidates each run
in seconds.
"""

import numpy as np
import pytest

from oracle import conv_ref

pytestmark = pytest.mark.gpu

# (row, batch): a 3x3 (Winograd + pairs), the 5x5 dominant shape, a 1x1, a first layer (space-to-depth), fc7
OPS = [(38, 2), (42, 1), (9, 2), (34, 1), (13, 3)]


@pytest.mark.parametrize("row,batch", OPS, ids=[f"row{r}-N{b}" for r, b in OPS])
def test_every_tuner_candidate_vs_oracle(cuda, row, batch):
    import torch

    from paper_1611_06945_b200 import corpus, runner, tuner
    from paper_1611_06945_b200.frontend import with_fused

    op = corpus.corpus(batch)[row]
    g = with_fused(op.graph(), "conv", "relu")
    node = g.node("conv")
    cands = tuner.candidates(node, g.edges)
    assert len(cands) >= 20
    tol = conv_ref.tolerance_for(op.in_chans * op.ksz * op.ksz)
    x, f, b = conv_ref.conv_inputs(op.batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz, f"cands:{row}:{batch}")
    want = conv_ref.ref_conv(x, f, b, op.stride, op.pad, relu=True)
    xs, fs, bs = conv_ref.conv_inputs(op.batch, op.in_chans, op.in_y, op.in_x, op.out_chans, op.ksz,
                                      f"cands-signed:{row}:{batch}", low=-1.0, high=1.0)
    pre = conv_ref.ref_conv(xs, fs, bs, op.stride, op.pad, relu=False).astype(np.float64)
    bound = 1e-5 * conv_ref.signed_bound(xs, fs, op.stride, op.pad) + 1e-6
    dev = [tuple(torch.from_numpy(a).cuda() for a in t) for t in ((x, f, b), (xs, fs, bs))]
    failures, kinds = [], set()
    for v, p in cands:
        plan = v.generate(node, g.edges, p)
        kinds.add((v.name, p.tma, p.cl))
        for which, (dx, dw, db) in enumerate(dev):
            cop = runner.ConvOp(plan, dx, dw, db)
            cop.y.fill_(float("nan"))
            cop.launch()
            torch.cuda.synchronize()
            got = cop.y.cpu().numpy()
            if which == 0:
                res = conv_ref.compare(got, want, tol)
                if not res.ok:
                    failures.append((v.name, p.to_string(), "reference data", res.max_rel_err))
            else:
                g64 = got.astype(np.float64)
                if not (np.abs(g64 - np.maximum(pre, 0.0)) <= bound).all() or (g64[pre < -bound] != 0.0).any():
                    failures.append((v.name, p.to_string(), "signed data"))
            del cop
    assert not failures, failures[:8]
    assert len(kinds) >= 3
