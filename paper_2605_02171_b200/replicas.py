"""Multi-GPU = replicas: every rank holds the whole index and
answers an independent slice of the query batch; the only exchange is the final
gather of k ids + scores per query (80 B/query at k=10), done once per batch
with torch.distributed (NCCL over NVLink on GPUs, gloo on CPU in tests).
Sharding the graph itself would change the traversal and break id parity.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(nq: int, world: int, rank: int):
    """Contiguous, balanced [lo, hi) slice of nq queries for `rank`."""
    base, extra = divmod(nq, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_results(ids: np.ndarray, scores: np.ndarray, counts: np.ndarray, nq: int,
                   device=None):
    """All-gather every rank's (ids, scores, counts) slice into full batch arrays
    in query order.  ids/scores: [n_local, k]; counts: [n_local]."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    k = ids.shape[1]
    dev = device or ("cuda" if dist.get_backend() == "nccl" else "cpu")
    sizes = [shard_bounds(nq, world, r) for r in range(world)]
    maxn = max(hi - lo for lo, hi in sizes)
    # pack [ids (k) | score bits (k) | count (1)] as int64 rows, padded to maxn
    pack = np.zeros((maxn, 2 * k + 1), np.int64)
    n = ids.shape[0]
    pack[:n, :k] = ids.astype(np.int64)
    pack[:n, k:2 * k] = scores.astype(np.float32).view(np.int32).astype(np.int64)
    pack[:n, 2 * k] = counts.astype(np.int64)
    t = torch.from_numpy(pack).to(dev)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    ids_all = np.empty((nq, k), np.uint32)
    sc_all = np.empty((nq, k), np.float32)
    cnt_all = np.empty(nq, np.uint32)
    for r, (lo, hi) in enumerate(sizes):
        blk = out[r].cpu().numpy()[: hi - lo]
        ids_all[lo:hi] = blk[:, :k].astype(np.uint32)
        sc_all[lo:hi] = blk[:, k:2 * k].astype(np.int32).view(np.float32)
        cnt_all[lo:hi] = blk[:, 2 * k].astype(np.uint32)
    return ids_all, sc_all, cnt_all


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist

    dev = device or ("cuda" if dist.get_backend() == "nccl" else "cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
