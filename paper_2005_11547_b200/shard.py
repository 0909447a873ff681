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
    return length_costs(np.diff(np.asarray(indptr, dtype=np.int64)), t)


def length_costs(lengths: np.ndarray, t: int) -> np.ndarray:
    return np.asarray(lengths, dtype=np.float64) * 3.0 + 2.0 * float(t)


def plan_shards(indptr, world: int, t: int = 1) -> np.ndarray:
    """Row boundaries (world+1,) of contiguous ranges with balanced cost."""
    return plan_shards_lengths(np.diff(np.asarray(indptr, dtype=np.int64)), world, t)


def plan_shards_lengths(lengths, world: int, t: int = 1) -> np.ndarray:
    """plan_shards from the row lengths alone (workloads.lengths gives them
    without generating the rows, so each rank can then generate only its own)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    cost = length_costs(lengths, t)
    n = cost.size
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


def minhash_host_multi(indptr, ids, weights, k: int, hashes, *, devices=None, bits: bool = False,
                       check: bool = True):
    """dart_minhash for a CSR batch in host memory, row-sharded over several
    GPUs driven by this one process.

    Each device sketches a contiguous, work-balanced row range through the
    host-buffer C entry point (dsk_minhash_csr_host: chunked copy-in /
    sketch / copy-out pipeline) and writes its rows straight into disjoint
    slices of the host outputs -- the "host gather", no collective.  One host
    thread per device (ctypes releases the GIL for the call).  Pinned input
    arrays give full PCIe overlap.

    Returns (values uint64[n, k], bits uint64[n, ceil(k/64)] or None,
    status int32[n]) as numpy arrays.
    """
    import ctypes
    from concurrent.futures import ThreadPoolExecutor

    from . import _lib
    from .api import raise_for_status
    from .constants import ValidationError, minhash_density
    if k < 1:
        raise ValidationError(f"k must be positive, got {k}")
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    n = indptr.size - 1
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = [int(d) for d in devices]
    words = (k + 63) // 64
    values = np.zeros((n, k), dtype=np.uint64)
    packed = np.zeros((n, words), dtype=np.uint64) if bits else None
    status = np.zeros(n, dtype=np.int32)
    bounds = plan_shards(indptr, len(devices), minhash_density(k))
    ctxs = [hashes.context(torch.device("cuda", d)) for d in devices]  # created up front
    lib = _lib.load()
    P = ctypes.c_void_p

    def run(r):
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        if r1 == r0:
            return 0
        e0 = int(indptr[r0])
        local = np.ascontiguousarray(indptr[r0:r1 + 1] - e0)
        with torch.cuda.device(devices[r]):
            return lib.dsk_minhash_csr_host(
                ctxs[r], P(local.ctypes.data), P(ids.ctypes.data + 8 * e0),
                P(weights.ctypes.data + 8 * e0), r1 - r0, k, P(values.ctypes.data + 8 * k * r0),
                P(packed.ctypes.data + 8 * words * r0) if bits else None,
                P(status.ctypes.data + 4 * r0), None, None)

    with ThreadPoolExecutor(max_workers=len(devices)) as pool:
        rcs = list(pool.map(run, range(len(devices))))
    for rc in rcs:
        _lib.check(rc, "dsk_minhash_csr_host")
    if check:
        raise_for_status(torch.from_numpy(status))
        repair_tied_rows(indptr, ids, weights, k, hashes, values, packed, status,
                         device=devices[0])
    return values, packed, status


def sharded_lsh(indptr, ids, weights, params, hashes, *, normalize: bool = False,
                group=None, gather: bool = False):
    """lsh_key + mix64 (ref/annindex.py:64-82, :135) for this rank's row range
    on this rank's GPU; ranges are balanced on the dart density t = L * K.

    Returns (bounds, LshBatch of the local rows[, gathered keys]).
    """
    from .api import lsh_batch
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    bounds = plan_shards(indptr, world, params.L * params.K)
    p, i, w = shard_csr(indptr, ids, weights, bounds, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    res = lsh_batch(p, i, w, params, hashes, normalize=normalize, device=dev)
    if gather and world > 1:
        return bounds, res, gather_rows(res.keys, bounds, group)
    return bounds, res


def lsh_host_multi(indptr, ids, weights, params, hashes, *, devices=None,
                   normalize: bool = False, check: bool = True):
    """(L, K) table keys for a CSR batch in host memory, row-sharded over
    several GPUs driven by this one process -- minhash_host_multi's
    counterpart for the LSH path (dsk_lsh_csr_host per device, each range
    written into its slice of the host outputs; no collective).

    Returns (keys uint64[n, L], status int32[n], phi int32[n]) as numpy arrays.
    """
    import ctypes
    from concurrent.futures import ThreadPoolExecutor

    from . import _lib
    from .api import DSK_STATUS_TIE, as_u64, lsh_batch, raise_for_status
    from .workloads import subset
    L, K = int(params.L), int(params.K)
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    n = indptr.size - 1
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = [int(d) for d in devices]
    keys = np.zeros((n, L), dtype=np.uint64)
    status = np.zeros(n, dtype=np.int32)
    phi = np.zeros(n, dtype=np.int32)
    bounds = plan_shards(indptr, len(devices), L * K)
    ctxs = [hashes.context(torch.device("cuda", d)) for d in devices]  # created up front
    lib = _lib.load()
    P = ctypes.c_void_p

    def run(r):
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        if r1 == r0:
            return 0
        e0 = int(indptr[r0])
        local = np.ascontiguousarray(indptr[r0:r1 + 1] - e0)
        with torch.cuda.device(devices[r]):
            return lib.dsk_lsh_csr_host(
                ctxs[r], P(local.ctypes.data), P(ids.ctypes.data + 8 * e0),
                P(weights.ctypes.data + 8 * e0), r1 - r0, L, K, int(bool(normalize)),
                P(keys.ctypes.data + 8 * L * r0), None, P(status.ctypes.data + 4 * r0),
                P(phi.ctypes.data + 4 * r0), None)

    with ThreadPoolExecutor(max_workers=len(devices)) as pool:
        rcs = list(pool.map(run, range(len(devices))))
    for rc in rcs:
        _lib.check(rc, "dsk_lsh_csr_host")
    if check:
        raise_for_status(torch.from_numpy(status))
        # rows with bit-identical ranks in a bucket: re-keyed by index tuple
        # through lsh_batch's tie path (ref/annindex.py:77-81)
        rows = np.nonzero((status & DSK_STATUS_TIE) != 0)[0]
        if rows.size:
            sp, si, sw = subset(indptr, ids, weights, rows)
            res = lsh_batch(sp, si, sw, params, hashes, normalize=normalize, stats=False,
                            device=torch.device("cuda", devices[0]))
            keys[rows] = as_u64(res.keys)
            status[rows] = res.status.cpu().numpy()
            phi[rows] = res.phi.cpu().numpy()
    return keys, status, phi


def repair_tied_rows(indptr, ids, weights, k: int, hashes, values, packed, status, *,
                     device=0) -> int:
    """Re-resolve host-path rows flagged DSK_STATUS_TIE by full index tuple.

    The C entry points order bit-identical ranks by fingerprint; the
    reference orders them by index tuple (ref/sketching.py:93-99).  Flagged
    rows are re-sketched through minhash_batch, whose tie path materialises
    their darts at phi* on the GPU and takes each bucket's minimum by
    (rank, element, nu, rho, w, r, j); the repaired rows overwrite `values`,
    `packed` and `status` in place.  Returns the number of rows repaired."""
    from .api import DSK_STATUS_TIE, as_u64, minhash_batch
    from .workloads import subset
    rows = np.nonzero((status & DSK_STATUS_TIE) != 0)[0]
    if rows.size == 0:
        return 0
    sp, si, sw = subset(indptr, ids, weights, rows)
    res = minhash_batch(sp, si, sw, k, hashes, values=values is not None,
                        bits=packed is not None, stats=False,
                        device=torch.device("cuda", int(device)))
    if values is not None:
        values[rows] = as_u64(res.values)
    if packed is not None:
        packed[rows] = as_u64(res.bits)
    status[rows] = res.status.cpu().numpy()
    return int(rows.size)
