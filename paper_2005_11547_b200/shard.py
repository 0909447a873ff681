"""Row sharding of a CSR batch across the GPUs of one node.

The sets of a batch are independent (every sketch depends only on (set,
seed, k)), so the multi-GPU path needs no collective on the
data path: each rank sketches a contiguous row range on its own GPU and the
results return by device-to-host copy.  Ranges are balanced by a per-row
work estimate (nnz plus a per-set term proportional to the dart density t:
a set costs ~2*t*phi areas plus a few regions per element).

`gather_rows` is an optional convenience for callers that want every row on
one process: a single all_gather over the process group (NCCL between GPUs,
gloo on CPU).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def row_costs(indptr: np.ndarray, t: int) -> np.ndarray:
    nnz = np.diff(np.asarray(indptr, dtype=np.int64))
    return nnz.astype(np.float64) * 3.0 + 2.0 * float(t)


def plan_shards(indptr, world: int, t: int = 1) -> np.ndarray:
    """Row boundaries (world+1,) of contiguous ranges with balanced cost."""
    if world < 1:
        raise ValueError("world must be >= 1")
    indptr = np.asarray(indptr, dtype=np.int64)
    n = indptr.size - 1
    cost = row_costs(indptr, t)
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    targets = cum[-1] * np.arange(1, world) / world
    cuts = np.searchsorted(cum, targets, side="left")
    bounds = np.concatenate([[0], np.clip(cuts, 0, n), [n]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


def shard_csr(indptr, ids, weights, bounds, rank: int):
    """Local CSR of rows [bounds[rank], bounds[rank+1]) with a rebased indptr."""
    indptr = np.asarray(indptr, dtype=np.int64)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    e0, e1 = int(indptr[r0]), int(indptr[r1])
    return indptr[r0:r1 + 1] - e0, ids[e0:e1], weights[e0:e1]


def gather_rows(local: torch.Tensor, bounds, group=None) -> torch.Tensor:
    """All ranks' row blocks concatenated in rank order (one all_gather)."""
    world = dist.get_world_size(group)
    sizes = [int(bounds[r + 1] - bounds[r]) for r in range(world)]
    mx = max(sizes) if sizes else 0
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)


def sharded_minhash(indptr, ids, weights, k: int, hashes, *, bits: bool = False,
                    group=None, gather: bool = False):
    """dart_minhash for this rank's row range on this rank's GPU.

    Returns (bounds, MinhashBatch of the local rows[, gathered values]).
    """
    from .api import minhash_batch
    from .constants import minhash_density
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    bounds = plan_shards(indptr, world, minhash_density(k))
    p, i, w = shard_csr(indptr, ids, weights, bounds, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    res = minhash_batch(p, i, w, k, hashes, bits=bits, device=dev)
    if gather and world > 1:
        return bounds, res, gather_rows(res.values, bounds, group)
    return bounds, res
