"""The unmodified reference package (`dartsketch`, pure Python + numpy) timed on
the host's cores: the CPU baseline BASELINE.md §2 names.

The package is installed, untouched, into `baseline/_ref` with

    python -m pip install --no-index --no-build-isolation --no-deps \
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>

(`--no-deps`: numpy is already in the image; the wheelhouse has no numpy
wheel to resolve).  `baseline/_ref` is git-ignored but travels to the GPU box
with the repository snapshot.  Nothing here is on the product path: bench.py
calls it only for its `cpu_baseline` leg and its `--impl reference` arm.

How it is timed (ref/bench.py:190-197): one worker process
per available core (`spawn`ed, single-threaded numpy), each given a
contiguous chunk of the same CSR rows the GPU consumed; every row becomes a
`WeightedSet.from_arrays` outside the timer, then the reference's own call
for the workload is timed with `time.perf_counter`:

  minhash workloads  dart_minhash(x, k, HashFamily(seed))  (+ one_bit for cfg3)
  cfg4 (LSH)         lsh_key(x, LshParams(L, K), h) and h.mix64(key) per table
                     (ref/annindex.py:64-82, :135)

Throughput = total sets / the slowest worker's busy time.
"""

from __future__ import annotations

import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(HERE, "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_PATH, "dartsketch"))


def _import_ref():
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import dartsketch
    return dartsketch


def _worker(job):
    """Runs in a spawned process: sketch rows [0, n) of the given CSR chunk."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np
    ds = _import_ref()
    kind, seed, k, L, K, onebit, indptr, ids, w = job
    h = ds.HashFamily(seed)
    sets = [ds.WeightedSet.from_arrays(ids[indptr[r]:indptr[r + 1]], w[indptr[r]:indptr[r + 1]])
            for r in range(indptr.size - 1)]
    out = np.zeros(len(sets), dtype=np.uint64)  # first value per row (sanity/parity probe)
    busy = 0.0
    if kind == "lsh":
        params = ds.LshParams(L, K)
        for r, x in enumerate(sets):
            t0 = time.perf_counter()
            keys = [h.mix64(key) for key in ds.lsh_key(x, params, h)]
            busy += time.perf_counter() - t0
            out[r] = keys[0]
    else:
        for r, x in enumerate(sets):
            t0 = time.perf_counter()
            sk = ds.dart_minhash(x, k, h)
            if onebit:
                ds.one_bit(sk)
            busy += time.perf_counter() - t0
            out[r] = sk.values[0]
    return busy, out


def cores() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class PyRefPool:
    """A pool of spawned workers that keep the reference imported between runs."""

    def __init__(self, workers: int | None = None):
        import multiprocessing as mp
        self.workers = workers or cores()
        self.pool = mp.get_context("spawn").Pool(self.workers)
        # import the reference in every worker up front (not timed)
        self.pool.map(_warm, range(self.workers))

    def close(self):
        self.pool.close()
        self.pool.join()

    def run(self, kind, seed, k, L, K, onebit, indptr, ids, w, rows):
        """Sketch rows [0, rows) split into contiguous per-worker chunks.

        Returns (sets/s, first value of every row as uint64[rows])."""
        import numpy as np
        bounds = np.linspace(0, rows, self.workers + 1).astype(np.int64)
        jobs = []
        for i in range(self.workers):
            r0, r1 = int(bounds[i]), int(bounds[i + 1])
            e0, e1 = int(indptr[r0]), int(indptr[r1])
            jobs.append((kind, seed, k, L, K, onebit, indptr[r0:r1 + 1] - e0, ids[e0:e1], w[e0:e1]))
        got = self.pool.map(_worker, jobs, chunksize=1)
        slowest = max(b for b, _ in got)
        firsts = np.concatenate([o for _, o in got]) if got else np.zeros(0, np.uint64)
        return rows / slowest if slowest > 0 else float("inf"), firsts

    def timed_sample(self, kind, seed, k, L, K, onebit, indptr, ids, w, seconds: float):
        """Size a sample to ~`seconds` of busy time per worker, then time it."""
        n = indptr.size - 1
        probe = min(n, 2 * self.workers)
        rate, _ = self.run(kind, seed, k, L, K, onebit, indptr, ids, w, probe)
        rows = int(min(n, max(probe, rate * seconds)))
        rate, firsts = self.run(kind, seed, k, L, K, onebit, indptr, ids, w, rows)
        return rate, rows, firsts


def _warm(_):
    _import_ref()
    return 0
