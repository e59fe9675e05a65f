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
