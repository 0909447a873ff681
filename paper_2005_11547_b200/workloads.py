"""Seeded synthetic CSR batches for the five BASELINE.json configurations.

The reference measures on synthetic sets only (PAPER.md:297-305,
ref/bench.py:82-100); BASELINE.json names five batch workloads.  This module
materialises each of them as CSR arrays (indptr int64[n+1], ids uint64[nnz],
weights float64[nnz]) that both the CUDA path and the CPU oracle consume.

Conventions:
  * data RNG = Generator(MT19937(SeedSequence(derive_seed(seed, 1, block)))),
    one stream per block of BLOCK_ROWS rows so any row range (a GPU shard)
    can be generated independently of how the batch is split;
    derive_seed restates ref/randomness.py:89-92;
  * distinct indices per set (duplicates are redrawn);
  * Uniform(0,1] = 1 - rng.random();
  * rows keep draw order.
"""

from __future__ import annotations

import dataclasses

import numpy as np

BLOCK_ROWS = 1 << 16


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    n: int
    d: int
    nnz: object          # int, or "zipf" for cfg5
    weights: str         # "uniform" | "exp_l1" | "lognormal1" | "lognormal2"
    seed: int
    kind: str            # "minhash" | "lsh"
    k: tuple = ()        # minhash slot counts
    L: int = 0
    K: int = 0
    onebit: bool = False
    description: str = ""


CONFIGS = {
    "cfg1": Workload("cfg1", 1000, 10_000, 256, "uniform", 0, "minhash", k=(64,),
                     description="1,000 sets, d=1e4, nnz=256, U(0,1], k=64, seed 0"),
    "cfg2": Workload("cfg2", 100_000, 1 << 20, 1024, "exp_l1", 1, "minhash", k=(256,),
                     description="1e5 sets, d=2^20, nnz=1024, Exp(1) with l1=1, k=256, seed 1"),
    "cfg3": Workload("cfg3", 1_000_000, 1 << 24, 64, "uniform", 2, "minhash",
                     k=(64, 256, 1024), onebit=True,
                     description="1e6 sets, d=2^24, nnz=64, U(0,1], k in {64,256,1024} + 1-bit, seed 2"),
    "cfg4": Workload("cfg4", 1_000_000, 1 << 24, 128, "lognormal1", 3, "lsh", L=100, K=20,
                     description="1e6 sets, d=2^24, nnz=128, LogNormal(0,1), (L,K)=(100,20), seed 3"),
    "cfg5": Workload("cfg5", 10_000_000, 1 << 26, "zipf", "lognormal2", 4, "minhash", k=(128,),
                     description="1e7 sets, d=2^26, nnz~Zipf(1.5) clipped [1,16384], "
                                 "LogNormal(0,2), k=128, seed 4"),
}


from .constants import derive_seed  # noqa: E402  (ref/randomness.py:89-92)


def _block_rng(seed: int, block: int) -> np.random.Generator:
    return np.random.Generator(np.random.MT19937(np.random.SeedSequence(
        derive_seed(seed, 1, block))))


def _distinct_rows(rng, d: int, lengths: np.ndarray) -> np.ndarray:
    """Concatenated rows of distinct ids in [0, d), one row per length."""
    total = int(lengths.sum())
    ids = rng.integers(0, d, size=total, dtype=np.uint64)
    starts = np.zeros(lengths.size + 1, dtype=np.int64)
    np.cumsum(lengths, out=starts[1:])
    # rows holding a repeated id (ascending), found by sorting within rows
    if lengths.size and (lengths == lengths[0]).all():
        srt = np.sort(ids.reshape(lengths.size, int(lengths[0])), axis=1)
        bad = np.flatnonzero((srt[:, 1:] == srt[:, :-1]).any(axis=1))
    else:
        row = np.repeat(np.arange(lengths.size, dtype=np.uint64), lengths)
        key = np.sort(row * np.uint64(d) + ids)
        bad = np.unique(key[1:][key[1:] == key[:-1]] // np.uint64(d)).astype(np.int64)
    for r in bad.tolist():  # rare: redraw the whole row without replacement
        a, b = starts[r], starts[r + 1]
        ids[a:b] = rng.choice(d, size=b - a, replace=False).astype(np.uint64)
    return ids


def _weights(rng, kind: str, lengths: np.ndarray) -> np.ndarray:
    total = int(lengths.sum())
    if kind == "uniform":
        return 1.0 - rng.random(total)
    if kind == "exp_l1":
        w = rng.standard_exponential(total)
        w = np.where(w > 0.0, w, np.finfo(np.float64).tiny)
        starts = np.zeros(lengths.size + 1, dtype=np.int64)
        np.cumsum(lengths, out=starts[1:])
        sums = np.add.reduceat(w, starts[:-1]) if total else np.zeros(0)
        return w / np.repeat(sums, lengths)
    if kind == "lognormal1":
        return rng.lognormal(0.0, 1.0, total)
    if kind == "lognormal2":
        return rng.lognormal(0.0, 2.0, total)
    raise ValueError(kind)


def _block_lengths(cfg: Workload, rng, rows: int) -> np.ndarray:
    """The row lengths of one block: the first draws of the block's stream."""
    if cfg.nnz == "zipf":
        return np.minimum(rng.zipf(1.5, size=rows), 16384).astype(np.int64)
    return np.full(rows, int(cfg.nnz), dtype=np.int64)


def _gen_block(cfg: Workload, block: int, rows: int):
    rng = _block_rng(cfg.seed, block)
    lengths = _block_lengths(cfg, rng, rows)
    if cfg.name == "cfg1":
        # d = 1e4 with nnz = 256: draw without replacement per set
        ids = np.concatenate([rng.choice(cfg.d, size=int(m), replace=False).astype(np.uint64)
                              for m in lengths.tolist()])
    else:
        ids = _distinct_rows(rng, cfg.d, lengths)
    w = _weights(rng, cfg.weights, lengths)
    return lengths, ids, w


def _block_rows(cfg: Workload, b: int) -> int:
    return min(BLOCK_ROWS, cfg.n - b * BLOCK_ROWS) if b * BLOCK_ROWS < cfg.n else BLOCK_ROWS


def lengths(cfg_name: str, n: int | None = None, start: int = 0) -> np.ndarray:
    """Row lengths (nnz) of rows [start, start + n) without generating the rows.

    Only the first draws of each block's stream are made (the lengths come
    first), so a shard plan over the full population (cfg5: 1e7 rows) costs
    about a second on the host."""
    cfg = CONFIGS[cfg_name]
    if n is None:
        n = cfg.n - start
    end = start + n
    if cfg.nnz != "zipf":
        return np.full(n, int(cfg.nnz), dtype=np.int64)
    out = []
    for b in range(start // BLOCK_ROWS, (end + BLOCK_ROWS - 1) // BLOCK_ROWS):
        rows = _block_rows(cfg, b)
        ln = _block_lengths(cfg, _block_rng(cfg.seed, b), rows)
        out.append(ln[max(start - b * BLOCK_ROWS, 0):min(end - b * BLOCK_ROWS, rows)])
    return np.concatenate(out) if out else np.zeros(0, np.int64)


# fork-inherited state of the block workers (one generate() call at a time)
_POOL_JOB = None


def _fill_block(task):
    """Generate one block and copy its requested rows into the shared outputs."""
    cfg, b, rows, lo, hi, e_out = task
    ids_out, w_out = _POOL_JOB
    ln, ids, w = _gen_block(cfg, b, rows)
    offs = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(ln, out=offs[1:])
    m = int(offs[hi] - offs[lo])
    ids_out[e_out:e_out + m] = ids[offs[lo]:offs[hi]]
    w_out[e_out:e_out + m] = w[offs[lo]:offs[hi]]
    return m


def _shared_empty(count: int, dtype) -> np.ndarray:
    import mmap
    nbytes = max(1, count * np.dtype(dtype).itemsize)
    return np.frombuffer(mmap.mmap(-1, nbytes), dtype=dtype, count=count)


def default_workers() -> int:
    import os
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def generate(cfg_name: str, n: int | None = None, start: int = 0, workers: int | None = None):
    """CSR arrays for rows [start, start + n) of a configuration.

    Blocks of BLOCK_ROWS rows have independent streams, so they are generated
    by a pool of forked host processes (`workers`, default: every core the
    process may use) writing straight into shared output arrays; the bytes do
    not depend on the worker count or on how the rows are split."""
    global _POOL_JOB
    cfg = CONFIGS[cfg_name]
    if n is None:
        n = cfg.n - start
    end = start + n
    lens = lengths(cfg_name, n, start)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    nnz = int(indptr[-1])
    b0, b1 = start // BLOCK_ROWS, (end + BLOCK_ROWS - 1) // BLOCK_ROWS
    tasks = []
    for b in range(b0, b1):
        rows = _block_rows(cfg, b)
        lo, hi = max(start - b * BLOCK_ROWS, 0), min(end - b * BLOCK_ROWS, rows)
        tasks.append((cfg, b, rows, lo, hi, int(indptr[b * BLOCK_ROWS + lo - start])))
    workers = min(workers or default_workers(), len(tasks))
    if workers > 1:
        import multiprocessing as mp
        ids, w = _shared_empty(nnz, np.uint64), _shared_empty(nnz, np.float64)
        _POOL_JOB = (ids, w)
        try:
            with mp.get_context("fork").Pool(workers) as pool:
                got = pool.map(_fill_block, tasks, chunksize=1)
        finally:
            _POOL_JOB = None
        ids, w = np.array(ids, copy=True), np.array(w, copy=True)  # private, writable
    else:
        ids, w = np.empty(nnz, np.uint64), np.empty(nnz, np.float64)
        _POOL_JOB = (ids, w)
        try:
            got = [_fill_block(t) for t in tasks]
        finally:
            _POOL_JOB = None
    assert sum(got) == nnz
    return indptr, ids, w


def subset(indptr, ids, w, rows):
    """CSR of the given row indices (in the given order)."""
    rows = np.asarray(rows, dtype=np.int64)
    lengths = indptr[rows + 1] - indptr[rows]
    out_ptr = np.zeros(rows.size + 1, dtype=np.int64)
    np.cumsum(lengths, out=out_ptr[1:])
    take = np.concatenate([np.arange(indptr[r], indptr[r + 1]) for r in rows.tolist()]) \
        if rows.size else np.zeros(0, np.int64)
    return out_ptr, np.ascontiguousarray(ids[take]), np.ascontiguousarray(w[take])
