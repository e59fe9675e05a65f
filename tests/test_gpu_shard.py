"""Multi-GPU path on the one-GPU test box: batch slabs computed
by separate ranks and gathered to rank 0 (shard.gather_to_root) are
bit-identical to the single-GPU run with the same kernel choice; and the
bench's N > 1 control flow (self-spawned ranks, per-unit slabs, gather, max
over ranks) runs end to end.

Both put every rank on cuda:0 with gloo collectives (NCCL refuses two ranks on
one GPU; gloo moves the slabs through host copies): a test of the code path
and of the bits, not a scaling number.
"""

import json
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(42, 20, "BN=128,sk=2,sw=0,dr=0,tm=1"), (38, 20, "BN=96,sk=4,sw=0,dr=0,tm=1"),
         (4, 20, "BN=32,sk=2,sw=0,dr=0,tm=3"), (41, 20, "BN=64,sk=1,sw=0,dr=0,tm=4"),
         (25, 20, "BN=32,sk=4,sw=1,dr=0,tm=1"), (34, 5, "BN=96,sk=1,sw=0,dr=0,tm=1")]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _op(row, batch, params):
    from paper_1611_06945_b200 import corpus
    from paper_1611_06945_b200.frontend import with_fused
    from paper_1611_06945_b200.variants import VARIANTS, TuneParams

    p = TuneParams.from_string("MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1," + params)
    op = corpus.corpus(batch)[row]
    g = with_fused(op.graph(), "conv", "relu")
    vname = "conv_fc" if row == 25 else ("conv_1x1" if op.ksz == 1 else "conv_umma")
    return op, g, VARIANTS[vname], p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_1611_06945_b200 import runner, shard
    from paper_1611_06945_b200.frontend import with_fused

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        items, local, full = [], {}, {}
        for u, (row, batch, params) in enumerate(CASES):
            op, g, v, p = _op(row, batch, params)
            node = g.node("conv")
            inputs = runner.node_test_inputs(node, g.edges, f"gather:{row}")
            x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
            if rank == 0:
                full[u] = torch.full(tuple(g.edges[node.outputs[0]].sizes), float("nan"), device="cuda")
            for r in range(world):
                first, count = shard.batch_slab(batch, world, r)
                items.append(shard.WorkItem(u, r, first, count))
                if r != rank:
                    continue
                gs = with_fused(op.with_batch(count).graph(), "conv", "relu")
                y = full[u][first:first + count] if rank == 0 else None
                o = runner.ConvOp(v.generate(gs.node("conv"), gs.edges, p), x[first:first + count].contiguous(), w, b, y=y)
                o.launch()
                local[len(items) - 1] = o.y
        torch.cuda.synchronize()
        dist.barrier()
        shard.gather_to_root(items, local, full, rank, stage_cpu=True)
        if rank == 0:
            out["full"] = {u: t.cpu() for u, t in full.items()}
    finally:
        dist.destroy_process_group()


def test_slabs_gathered_to_root_bit_identical(cuda):
    from paper_1611_06945_b200 import runner

    world = 3
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    for u, (row, batch, params) in enumerate(CASES):
        op, g, v, p = _op(row, batch, params)
        node = g.node("conv")
        inputs = runner.node_test_inputs(node, g.edges, f"gather:{row}")
        x, w, b = (runner.to_device(inputs[e]) for e in node.inputs)
        whole = runner.ConvOp(v.generate(node, g.edges, p), x, w, b)
        whole.launch()
        torch.cuda.synchronize()
        assert torch.equal(out["full"][u], whole.y.cpu()), (row, batch, params)


def test_bench_two_ranks_shard_mode_control_flow(cuda):
    env = dict(os.environ, B2C_BENCH_ONE_GPU_TEST="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--no-cpu"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    mg = line["multi_gpu"]
    assert mg["gather"] and mg["gather_inclusive_ms"] >= mg["compute_only_ms"] > 0
    assert line["config"]["flops_per_step"] == 152691710080  # the whole sweep, split over the ranks
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0  # host-buffer path on both ranks
