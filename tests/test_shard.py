"""Multi-GPU partitioning logic and the output gather,
exercised with world_size 2 over gloo on CPU (the GPU path runs the same
functions over NCCL)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_06945_b200.shard import batch_slab, gather_batch, lpt_assign


def test_batch_slabs_cover_and_balance():
    assert [batch_slab(20, 8, r) for r in range(8)] == [(0, 3), (3, 3), (6, 3), (9, 3), (12, 2), (14, 2), (16, 2), (18, 2)]
    for n in (1, 5, 20, 7):
        for world in (1, 2, 4, 8):
            slabs = [batch_slab(n, world, r) for r in range(world)]
            assert sum(c for _, c in slabs) == n
            assert max(c for _, c in slabs) - min(c for _, c in slabs) <= 1
            pos = 0
            for first, count in slabs:
                assert first == pos
                pos += count
    with pytest.raises(ValueError):
        batch_slab(5, 2, 2)


def test_lpt_assign_balances_sweep_costs():
    from paper_1611_06945_b200 import corpus

    costs = [op.flops_computed for _, op in corpus.sweep_ops([1, 5, 20])]
    for world in (2, 4, 8):
        parts = lpt_assign(costs, world)
        assert sorted(i for p in parts for i in p) == list(range(len(costs)))
        loads = [sum(costs[i] for i in p) for p in parts]
        # LPT bound: max load <= mean + largest unit
        assert max(loads) <= sum(costs) / world + max(costs)
    assert lpt_assign([3.0, 1.0, 2.0], 2) == [[0], [1, 2]]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_total, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        first, count = batch_slab(n_total, world, rank)
        # each rank "computes" its slab of an NCHW output: image i holds value i
        y = torch.arange(first, first + count, dtype=torch.float32).view(count, 1, 1, 1).expand(count, 3, 2, 2).contiguous()
        full = gather_batch(y, n_total)
        results[rank] = full.clone()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [5, 20, 1])
def test_gather_batch_gloo_world2(n_total):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n_total, results), nprocs=world, join=True)
    want = torch.arange(n_total, dtype=torch.float32).view(n_total, 1, 1, 1).expand(n_total, 3, 2, 2)
    for r in range(world):
        assert torch.equal(results[r], want)


def test_bench_reference_arm_runs_on_cpu():
    """The driver's reference arm (bench.py --impl reference) needs no GPU: the
    oracle port timed on host cores, one JSON line from rank 0, silent other ranks."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
           "--batches", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "TFLOP/s"
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""
