"""Multi-GPU plumbing: pairs shard across ranks; NCCL only gathers results.

Two ways to split a batch: fixed shards (the default: a deterministic LPT partition of
the batch over nominal cells, lpt_partition; shard_range / split_range
give contiguous ranges) or cross-GPU dynamic balancing (NEXT #1): every rank holds the whole batch and
its persistent kernel claims pairs from one counter in rank 0's HBM with system-scope
atomics (agatha_queue_*, handle exchanged by share_queue_handle); each rank's output has
only its own rows, merged by merge_claimed.

The path has no data exchange between pairs (§5.8 l.843-846: independent
per-GPU processing), so each rank aligns its own shard and the only collective is the
gather of the fixed 24-byte result records (BASELINE.json north_star: "NCCL over
NVLink used only to gather results").  Shards are contiguous ranges of the counter-
based pair stream, so every rank can generate its own inputs (synth/).

This module is plumbing: it never touches sequences or scores.
"""
from __future__ import annotations

from typing import Tuple

RECORD_BYTES = 24


def shard_range(pairs_per_rank: int, rank: int) -> Tuple[int, int]:
    """Weak scaling: rank r owns pairs [r*n, (r+1)*n) of the stream."""
    return rank * pairs_per_rank, (rank + 1) * pairs_per_rank


def split_range(n_pairs: int, world: int, rank: int) -> Tuple[int, int]:
    """Strong scaling: a fixed batch of n_pairs split into contiguous near-equal shards."""
    base, extra = divmod(n_pairs, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def nominal_cells(m, n, band_left: int, band_right: int):
    """Nominal in-band in-table cells of un-terminated pairs (the work estimate of
    SURVEY.md §8(a2), [A.3]): #{(i, j) : 1 <= i <= m, 1 <= j <= n, -bl <= i - j <= br},
    vectorised over numpy arrays m, n; a negative band side is unbounded.  Computed as
    m*n minus the two triangles outside the band:
      #{i - j > br} = sum_{j=1..n} max(0, m - br - j),
      #{j - i > bl} = sum_{i=1..m} max(0, n - bl - i)."""
    import numpy as np

    m = np.asarray(m, np.int64)
    n = np.asarray(n, np.int64)

    def tri(k, cnt):  # sum_{x=1..cnt} max(0, k - x)
        t = np.clip(np.minimum(cnt, k - 1), 0, None)
        return t * k - t * (t + 1) // 2

    out = m * n
    if band_right >= 0:
        out = out - tri(m - band_right, n)
    if band_left >= 0:
        out = out - tri(n - band_left, m)
    return out


def lpt_partition(weights, world: int):
    """Deterministic LPT (longest processing time first) partition of items with the given
    weights (nominal cells) into `world` shards: items in descending
    weight (ties: lower index first) each go to the currently lightest shard (ties: lower
    rank).  Returns one ascending index array per rank.  Every shard's load is within the
    largest single weight of every other shard's."""
    import heapq

    import numpy as np

    w = np.asarray(weights, np.int64)
    if world == 1:
        return [np.arange(len(w), dtype=np.int64)]
    order = np.lexsort((np.arange(len(w)), -w))
    heap = [(0, r) for r in range(world)]
    owner = np.empty(len(w), np.int64)
    wl = w[order].tolist()
    for k, wk in zip(order.tolist(), wl):
        load, r = heapq.heappop(heap)
        owner[k] = r
        heapq.heappush(heap, (load + wk, r))
    return [np.nonzero(owner == r)[0] for r in range(world)]


def scatter_gathered(gathered_rows, shards, n_total: int):
    """Rows gathered from the ranks (rank r's shard padded to the largest shard, in rank
    order) back into stream order: row t of rank r is pair shards[r][t]."""
    import numpy as np

    pad = max(len(s) for s in shards)
    out = np.zeros(n_total, gathered_rows.dtype)
    for r, s in enumerate(shards):
        out[s] = gathered_rows[r * pad:r * pad + len(s)]
    return out


def share_queue_handle(handle: bytes, world: int, src: int = 0) -> bytes:
    """Broadcast the 64-byte CUDA IPC handle of rank src's shared pair counter
    (agatha_queue_create) to every rank; the others map it with agatha_queue_open."""
    import torch.distributed as dist

    if world == 1:
        return handle
    box = [handle]
    dist.broadcast_object_list(box, src=src)
    return bytes(box[0])


def merge_claimed(records, world: int, group=None):
    """Merge per-rank result buffers in which each rank filled only the rows it claimed
    (all other rows zero): an all_reduce(SUM) over the records viewed as int64 words, which
    is exact because every row is non-zero on at most one rank."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.all_reduce(records.view(-1).view(torch.int64), op=dist.ReduceOp.SUM, group=group)
    return records


def gather_results(local, world: int, group=None):
    """all_gather the ranks' result buffers (uint8 tensors of 24*n bytes, same n on every
    rank: shards of unequal size are padded to the largest) into one tensor in rank order.
    NCCL on CUDA tensors, gloo on CPU tensors."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    out = torch.empty(local.numel() * world, dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)
    else:  # gloo (CPU tests, or the one-GPU test mode of bench.py): list form
        dist.all_gather(list(out.chunk(world)), local, group=group)
    return out


def max_over_ranks(value: float, device, world: int) -> float:
    """The slowest rank's time (the job's time)."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def sum_over_ranks(value: float, device, world: int) -> float:
    import torch
    import torch.distributed as dist

    if world == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t[0])
