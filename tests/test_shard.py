"""Multi-GPU partitioning logic and the output gather,
exercised with world_size 2 over gloo on CPU (the GPU path runs the same
functions over NCCL)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_06945_b200.shard import WorkItem, batch_slab, gather_batch, gather_to_root, lpt_assign, plan_sweep


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
    reference's own ref_conv (baseline/_ref; the oracle port when that is not
    installed) timed on host cores, one JSON line from rank 0, silent other ranks."""
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
    ref_installed = os.path.isdir(os.path.join(root, "baseline", "_ref", "site", "cuclgen"))
    assert line["cpu_baseline"]["kind"] == ("reference" if ref_installed else "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["config"]["ops_per_step"] == 43
    assert line["cpu_baseline"]["cores"] >= 1 and line["cpu_baseline"]["cpu_model"]
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_plan_sweep_covers_every_image_once_and_balances():
    from paper_1611_06945_b200 import corpus

    sweep = corpus.sweep_ops([1, 5, 20])
    batches = [op.batch for _, op in sweep]
    costs = [op.flops_computed / op.batch for _, op in sweep]
    for world in (1, 2, 4, 8):
        items = plan_sweep(batches, world, lambda u, c: costs[u] * c)
        for u, b in enumerate(batches):
            mine = sorted((it.first, it.count) for it in items if it.unit == u)
            pos = 0
            for first, count in mine:  # contiguous, disjoint, complete
                assert first == pos and count >= 1
                pos += count
            assert pos == b
            if b >= world:  # north_star config 5: one batch_slab per rank (20 over 8 -> 3,3,3,3,2,2,2,2)
                mine_u = [it for it in items if it.unit == u]
                assert [it.count for it in mine_u] == [batch_slab(b, world, k)[1] for k in range(world)]
                assert sorted(it.rank for it in mine_u) == list(range(world))
        loads = [sum(costs[it.unit] * it.count for it in items if it.rank == r) for r in range(world)]
        assert max(loads) <= sum(loads) / world + max(costs)  # LPT bound
        assert items == plan_sweep(batches, world, lambda u, c: costs[u] * c)  # deterministic
    assert [(it.rank, it.count) for it in plan_sweep([20], 8)] == [(r, 3 if r < 4 else 2) for r in range(8)]
    assert [(it.rank, it.count) for it in plan_sweep([20, 20], 8)][8:] == [(r, 3 if r >= 4 else 2) for r in
                                                                            (4, 5, 6, 7, 0, 1, 2, 3)]


def _p2p_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batches = [20, 5, 1, 3]
        items = plan_sweep(batches, world)
        full = {u: torch.full((b, 2, 3, 3), -1.0) for u, b in enumerate(batches)} if rank == 0 else {}
        local = {}
        for i, it in enumerate(items):
            if it.rank != rank:
                continue
            # image j of unit u holds 100*u + j, computed by its owner
            y = (100.0 * it.unit + torch.arange(it.first, it.first + it.count, dtype=torch.float32)).view(-1, 1, 1, 1)
            y = y.expand(it.count, 2, 3, 3).contiguous()
            if rank == 0:
                full[it.unit][it.first: it.first + it.count].copy_(y)
            local[i] = y
        dist.barrier()
        for w in gather_to_root(items, local, full, rank):
            w.wait()
        if rank == 0:
            results["full"] = {u: t.clone() for u, t in full.items()}
    finally:
        dist.destroy_process_group()


def test_gather_to_root_gloo_world3():
    """Every slab computed off rank 0 lands in place in rank 0's full outputs."""
    world = 3
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_p2p_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for u, b in enumerate([20, 5, 1, 3]):
        want = (100.0 * u + torch.arange(b, dtype=torch.float32)).view(-1, 1, 1, 1).expand(b, 2, 3, 3)
        assert torch.equal(results["full"][u], want)


def test_bench_spawns_ranks_for_gpus_flag(monkeypatch):
    """bench.py --gpus N without WORLD_SIZE re-launches itself under torch.distributed.run."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench

    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    monkeypatch.setattr(subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0
    cmd = calls[0]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"] and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
