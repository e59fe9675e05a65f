"""Multi-GPU partitioning of the conv sweep.

The path shards with no exchange during compute:

* by batch: images are independent, so an op's N images are split into
  contiguous slabs, one per rank (20 images over 8 GPUs -> 3,3,3,3,2,2,2,2);
  filters and bias are replicated (regenerated per rank from the same seed);
* by op: the sweep's ops are independent units, assigned longest-processing-
  time first by their roofline time.

The only collective is the optional output gather to one rank (north_star:
"NCCL over NVLink used only to gather outputs"): an NCHW slab of images is a
contiguous block, so gathering is a concatenation along dim 0.  Uneven slabs
are padded to the largest slab for ``all_gather`` and trimmed afterwards.
The functions take a ``torch.distributed`` process group, so they run over
NCCL on GPUs and over gloo in the CPU tests.
"""

from __future__ import annotations

import heapq


def batch_slab(n: int, world: int, rank: int) -> tuple:
    """(first image, image count) of `rank`'s contiguous slab of `n` images;
    the first n % world ranks get one extra image."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError(f"bad slab request n={n} world={world} rank={rank}")
    base, extra = divmod(n, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def lpt_assign(costs, world: int) -> list:
    """Longest-processing-time-first assignment of independent units (e.g. the
    sweep's ops, costed by roofline time) to `world` ranks; returns a list of
    unit-index lists, one per rank.  Deterministic (ties by unit index, rank)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    for lst in out:
        lst.sort()
    return out


def gather_batch(y_local, n_total: int, group=None, dst_all: bool = True):
    """Concatenate every rank's output slab (dim 0 = images, NCHW) into the
    full batch of `n_total` images.  Collective over `group`; with dst_all the
    result is returned on every rank (all_gather), else only rank 0's return
    value is meaningful."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = [batch_slab(n_total, world, r)[1] for r in range(world)]
    cmax = max(counts)
    shape = (cmax,) + tuple(y_local.shape[1:])
    padded = torch.zeros(shape, dtype=y_local.dtype, device=y_local.device)
    padded[: y_local.shape[0]].copy_(y_local)
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


# ----------------------------------------------------------------------------- sweep partition + gather


class WorkItem:
    """One rank's share of one sweep unit (op at a batch size): images
    [first, first + count) of the unit's batch, run on ``rank``."""

    __slots__ = ("unit", "rank", "first", "count")

    def __init__(self, unit: int, rank: int, first: int, count: int):
        self.unit, self.rank, self.first, self.count = unit, rank, first, count

    def __repr__(self):
        return f"WorkItem(unit={self.unit}, rank={self.rank}, first={self.first}, count={self.count})"

    def __eq__(self, other):
        return isinstance(other, WorkItem) and (self.unit, self.rank, self.first, self.count) == (
            other.unit, other.rank, other.first, other.count)


def plan_sweep(batch_sizes, world: int, cost=None) -> list:
    """Strong-scaling partition of the sweep's units over
    ``world`` ranks, identical on every rank (deterministic):

    * a unit whose batch is >= world is cut into ``world`` contiguous slabs
      (batch_slab: 20 images over 8 GPUs -> 3,3,3,3,2,2,2,2), one per rank; when
      the slabs are uneven the larger ones go to the least-loaded ranks (so the
      extra images rotate over the ranks from unit to unit);
    * a smaller batch is cut into single images (a batch-1 unit stays whole)
      and those pieces go longest-first to the least-loaded rank (LPT over the
      load the slabs already put on each rank).

    ``cost(unit, count)`` estimates a piece's time (default: its image count).
    Returns WorkItems ordered by unit, then first image."""
    cost = cost or (lambda unit, count: float(count))
    items, loads = [], [0.0] * world
    small = []
    for u, b in enumerate(batch_sizes):
        if b >= world:
            by_load = sorted(range(world), key=lambda k: (loads[k], k))
            for k in range(world):  # slab k (the larger ones first) -> k-th least-loaded rank
                first, count = batch_slab(b, world, k)
                r = by_load[k]
                items.append(WorkItem(u, r, first, count))
                loads[r] += cost(u, count)
        else:
            small.extend((u, i, 1) for i in range(b))
    for u, first, count in sorted(small, key=lambda p: (-cost(p[0], p[2]), p[0], p[1])):
        r = min(range(world), key=lambda k: (loads[k], k))
        items.append(WorkItem(u, r, first, count))
        loads[r] += cost(u, count)
    items.sort(key=lambda it: (it.unit, it.first))
    return items


def gather_to_root(items, local_out: dict, full_out: dict, rank: int, group=None, stage_cpu: bool = False):
    """Move every slab computed off rank 0 into rank 0's full output tensors:
    point-to-point sends (owner -> 0) and receives (0 <- owner) of the
    contiguous NCHW slabs, issued as one batch (NCCL groups them; they run on
    NCCL's stream after the work already queued on the current stream, so the
    transfers overlap whatever the caller queues next).

    ``items``: the same WorkItem list on every rank (a group of the sweep);
    ``local_out[i]``: this rank's output slab for items[i] (owner ranks);
    ``full_out[unit]``: rank 0's full output of a unit (images on dim 0).
    Returns the async works (wait() them before reading full_out).  With
    ``stage_cpu`` (gloo, which cannot send CUDA tensors) the transfers are
    synchronous through host copies."""
    import torch.distributed as dist

    ops, post = [], []
    for i, it in enumerate(items):
        if it.rank == 0:
            continue
        if rank == it.rank:
            t = local_out[i]
            ops.append(dist.P2POp(dist.isend, t.cpu() if stage_cpu else t, 0, group))
        elif rank == 0:
            dst = full_out[it.unit][it.first: it.first + it.count]
            if stage_cpu:
                buf = dst.cpu()
                ops.append(dist.P2POp(dist.irecv, buf, it.rank, group))
                post.append((dst, buf))
            else:
                ops.append(dist.P2POp(dist.irecv, dst, it.rank, group))
    if not ops:
        return []
    works = dist.batch_isend_irecv(ops)
    if stage_cpu:
        for w in works:
            w.wait()
        for dst, buf in post:
            dst.copy_(buf)
        return []
    return works
