"""Measurement of the SURVEY.md §8(f) rows built after the hot path.

    python bench_next.py [--row bottomk|lshindex|dsk1|all]

One JSON line per row, with bench.py's timing rules: >= 3 warm-up calls,
device-resident inputs timed with CUDA events on the launching stream (host
APIs timed by wall clock around the synchronous call), and the C oracle
port of the reference on a bounded sample as the CPU baseline
(`cpu_baseline.kind` "port"; the oracle is the checker, never the product).

  bottomk   bottom_k (ref/sketching.py:146-156) for cfg3 rows (nnz 64), k = 64:
            sketches/s through bottom_k_batch (K6 enumeration + device lexsort).
  lshindex  LshIndex (ref/annindex.py:85-158) on cfg4 rows, L = 100, K = 20:
            bulk insert (points/s) and query_many (queries/s).  The CPU arm is a
            port of the index around the oracle's lsh_csr; its answers are
            checked against the GPU index on the first queries.
  dsk1      DSK1 minhash records (ref/sketching.py:210-231), k = 256: the
            record kernel (GB/s against the HBM peak) and dump_sketches with
            the bytes on the host.
  icws      the ICWS comparator (ref/baselines.py:84-161), cfg3 rows, k = 64.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)


def _events_ms(fn, steps=3, warmup=3):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def _dev_csr(indptr, ids, w, dev):
    import torch
    return (torch.from_numpy(indptr).to(dev), torch.from_numpy(ids.view(np.int64)).to(dev),
            torch.from_numpy(w).to(dev))


def row_bottomk(dev):
    from oracle.oracle import Oracle
    from paper_2005_11547_b200 import HashFamily, bottom_k_batch, workloads
    n, k = 100_000, 64
    indptr, ids, w = workloads.generate("cfg3", n=n)
    fam = HashFamily(2)
    p, i, ww = _dev_csr(indptr, ids, w, dev)
    ms = _events_ms(lambda: bottom_k_batch(p, i, ww, k, fam, check=False))
    orc = Oracle(2)
    t0, rows = time.perf_counter(), 0
    while time.perf_counter() - t0 < 5.0 and rows < n:
        a, b = indptr[rows], indptr[rows + 1]
        orc.bottom_k(ids[a:b], w[a:b], k)
        rows += 1
    cdt = time.perf_counter() - t0
    return {"row": "bottom_k", "metric": "sketches/sec", "value": n / (ms / 1e3),
            "unit": "sketches/sec", "ms_per_step": ms,
            "config": {"workload": "cfg3 rows", "sets": n, "nnz": 64, "k": k, "t": k},
            "cpu_baseline": {"value": rows / cdt, "unit": "sketches/sec", "cores": 1,
                             "kind": "port",
                             "sample": f"first {rows} sets, oracle bottom_k, 1 thread"}}


class CpuLshIndex:
    """Port of LshIndex (ref/annindex.py:85-158) around the oracle's keys."""

    def __init__(self, orc, L, K, j1):
        self.orc, self.L, self.K, self.j1 = orc, L, K, j1
        self.tables = {}
        self.sets = []

    def insert_many(self, indptr, ids, w):
        keys, _, st, _, _ = self.orc.lsh_csr(indptr, ids, w, self.L, self.K, normalize=True)
        assert (st == 0).all()
        for r in range(indptr.size - 1):
            a, b = indptr[r], indptr[r + 1]
            pid = len(self.sets)
            order = np.argsort(ids[a:b], kind="stable")
            self.sets.append((ids[a:b][order], w[a:b][order]))
            c = math.frexp(float(np.sum(w[a:b])))[1] - 1
            for tbl, key in enumerate(keys[r].tolist()):
                self.tables.setdefault((c, tbl, key), []).append(pid)

    @staticmethod
    def _jaccard(x, y):
        (xi, xw), (yi, yw) = x, y
        u = np.union1d(xi, yi)
        xa = np.zeros(u.size)
        ya = np.zeros(u.size)
        xa[np.searchsorted(u, xi)] = xw
        ya[np.searchsorted(u, yi)] = yw
        mn, mx = 0.0, 0.0
        for p, q in zip(xa.tolist(), ya.tolist()):  # ascending ids, as ref/core.py:103-120
            mn += min(p, q)
            mx += max(p, q)
        return mn / mx

    def query_many(self, indptr, ids, w):
        rows, classes = [], []
        present = {c for (c, _, _) in self.tables}
        for r in range(indptr.size - 1):
            l1 = float(np.sum(w[indptr[r]:indptr[r + 1]]))
            lo, hi = self.j1 * l1, l1 / self.j1
            c = math.frexp(lo)[1] - 1
            while math.ldexp(1.0, c) < hi:
                if c in present:
                    rows.append(r)
                    classes.append(c)
                c += 1
        if not rows:
            return [[] for _ in range(indptr.size - 1)]
        lens = np.array([indptr[r + 1] - indptr[r] for r in rows])
        sp = np.zeros(len(rows) + 1, dtype=np.int64)
        np.cumsum(lens, out=sp[1:])
        si = np.concatenate([ids[indptr[r]:indptr[r + 1]] for r in rows])
        sw = np.concatenate([np.ldexp(w[indptr[r]:indptr[r + 1]], -c)
                             for r, c in zip(rows, classes)])
        keys, _, st, _, _ = self.orc.lsh_csr(sp, si, sw, self.L, self.K)
        cand = [set() for _ in range(indptr.size - 1)]
        for q, (r, c) in enumerate(zip(rows, classes)):
            for tbl, key in enumerate(keys[q].tolist()):
                cand[r].update(self.tables.get((c, tbl, key), ()))
        out = []
        for r in range(indptr.size - 1):
            a, b = indptr[r], indptr[r + 1]
            order = np.argsort(ids[a:b], kind="stable")
            qx = (ids[a:b][order], w[a:b][order])
            res = [(pid, self._jaccard(qx, self.sets[pid])) for pid in cand[r]]
            res.sort(key=lambda item: (-item[1], item[0]))
            out.append(res)
        return out


def row_lshindex(dev):
    import torch
    from oracle.oracle import Oracle
    from paper_2005_11547_b200 import HashFamily, LshIndex, LshParams, WeightedSet, workloads
    n_pts, n_q = 100_000, 1_000
    L, K, j1 = 100, 20, 0.5
    indptr, ids, w = workloads.generate("cfg4", n=n_pts)
    qp, qi, qw = workloads.generate("cfg4", n=n_q // 2, start=n_pts)
    # half the queries are indexed points (exact matches), half unseen sets
    sp, si, sw = workloads.subset(indptr, ids, w, np.arange(0, n_pts, n_pts // (n_q // 2)))
    qp = np.concatenate([sp, qp[1:] + sp[-1]])
    qi = np.concatenate([si, qi])
    qw = np.concatenate([sw, qw])

    def sets_of(p_, i_, w_):
        return [WeightedSet.from_arrays(i_[p_[r]:p_[r + 1]], w_[p_[r]:p_[r + 1]])
                for r in range(p_.size - 1)]
    pts, qs = sets_of(indptr, ids, w), sets_of(qp, qi, qw)
    fam = HashFamily(3)
    params = LshParams(L, K, j1)
    LshIndex(params, fam, device=dev).insert_many(range(1000), pts[:1000])  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    idx = LshIndex(params, fam, device=dev)
    idx.insert_many(range(n_pts), pts)
    idx._build_tables()
    torch.cuda.synchronize()
    t_ins = time.perf_counter() - t0
    idx.query_many(qs[:50])
    t0 = time.perf_counter()
    got = idx.query_many(qs)
    t_q = time.perf_counter() - t0
    # CPU port: inserts on all threads (keys), queries on a bounded sample
    orc = Oracle(3)
    cpu = CpuLshIndex(orc, L, K, j1)
    t0 = time.perf_counter()
    cpu.insert_many(indptr, ids, w)
    c_ins = time.perf_counter() - t0
    nq_cpu = 40
    qsp, qsi, qsw = workloads.subset(qp, qi, qw, np.r_[0:nq_cpu // 2, n_q // 2:n_q // 2 + nq_cpu // 2])
    t0 = time.perf_counter()
    cres = cpu.query_many(qsp, qsi, qsw)
    c_q = time.perf_counter() - t0
    sel = list(range(nq_cpu // 2)) + list(range(n_q // 2, n_q // 2 + nq_cpu // 2))
    agree = all([(int(p), s) for p, s in got[q]] == cres[j] for j, q in enumerate(sel))
    from oracle.oracle import default_threads
    return [
        {"row": "LshIndex.insert", "metric": "points/sec", "value": n_pts / t_ins,
         "unit": "points/sec", "ms_per_step": t_ins * 1e3,
         "config": {"workload": "cfg4 rows", "points": n_pts, "L": L, "K": K},
         "cpu_baseline": {"value": n_pts / c_ins, "unit": "points/sec",
                          "cores": default_threads(), "kind": "port",
                          "sample": f"all {n_pts} points (oracle keys on all threads + dict tables)"}},
        {"row": "LshIndex.query", "metric": "queries/sec", "value": n_q / t_q,
         "unit": "queries/sec", "ms_per_step": t_q * 1e3,
         "config": {"workload": "cfg4 rows", "points": n_pts, "queries": n_q, "L": L, "K": K,
                    "j1": j1, "mean_results_per_query": float(np.mean([len(r) for r in got]))},
         "cpu_baseline": {"value": nq_cpu / c_q, "unit": "queries/sec", "cores": default_threads(),
                          "kind": "port",
                          "sample": f"{nq_cpu} queries (half indexed, half unseen)"},
         "cpu_gpu_results_identical": bool(agree)},
    ]


def row_dsk1(dev):
    import torch
    from paper_2005_11547_b200 import _lib, dump_sketches
    from paper_2005_11547_b200.api import _ptr, _stream_ptr
    n, k, seed = 200_000, 256, 2
    rng = np.random.default_rng(5)
    vals = torch.from_numpy(rng.integers(-2**63, 2**63 - 1, size=(n, k), dtype=np.int64)).to(dev)
    rec = 20 + 8 * k
    out = torch.empty(n * rec, dtype=torch.uint8, device=dev)
    lib = _lib.load()

    def kern():
        _lib.check(lib.dsk_dsk1_records(1, k, seed, _ptr(vals), n, _ptr(out), _stream_ptr(dev)),
                   "dsk_dsk1_records")
    ms = _events_ms(kern)
    moved = n * rec + n * 8 * k
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6543.1) \
        if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else 6543.1
    for _ in range(2):  # warm: the pinned staging block is cached after first use
        dump_sketches(vals, 1, k, seed)
    t0 = time.perf_counter()
    blob = dump_sketches(vals, 1, k, seed)
    t_api = time.perf_counter() - t0
    # CPU port of dump_sketch (ref/sketching.py:224-231), vectorised with numpy
    host = vals.cpu().numpy()
    t0 = time.perf_counter()
    dt = np.dtype([("magic", "S4"), ("ver", "u1"), ("kind", "u1"), ("res", "<u2"), ("k", "<u4"),
                   ("seed", "<u8"), ("payload", "<u8", (k,))])
    arr = np.empty(n, dtype=dt)
    arr["magic"] = b"DSK1"
    arr["ver"] = 1
    arr["kind"] = 1
    arr["res"] = 0
    arr["k"] = k
    arr["seed"] = seed
    arr["payload"] = host.view(np.uint64)
    cblob = arr.tobytes()
    c_dt = time.perf_counter() - t0
    assert cblob == blob
    return {"row": "DSK1 records", "metric": "records/sec", "value": n / (ms / 1e3),
            "unit": "records/sec", "ms_per_step": ms,
            "config": {"kind": "minhash", "k": k, "records": n, "record_bytes": rec},
            "roofline": {"bound": "hbm", "achieved": moved / (ms / 1e3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": moved / (ms / 1e3) / 1e9 / peak},
            "e2e": {"value": n / t_api, "unit": "records/sec",
                    "api": "dump_sketches (bytes on the host)",
                    "d2h_bytes_per_step": n * rec},
            "cpu_baseline": {"value": n / c_dt, "unit": "records/sec", "cores": 1, "kind": "port",
                             "sample": f"{n} records, numpy structured array"},
            "cpu_gpu_bytes_identical": True}


def row_icws(dev):
    from oracle.oracle import Oracle
    from paper_2005_11547_b200 import HashFamily, icws_batch, workloads
    n, k = 100_000, 64
    indptr, ids, w = workloads.generate("cfg3", n=n)
    fam = HashFamily(2)
    p, i, ww = _dev_csr(indptr, ids, w, dev)
    ms = _events_ms(lambda: icws_batch(p, i, ww, k, fam, check=False))
    # CPU: the reference's numpy formulation (ref/baselines.py:106-136) over
    # the oracle's hash, one set at a time, single thread
    orc = Oracle(2)
    t0, rows = time.perf_counter(), 0
    while time.perf_counter() - t0 < 5.0 and rows < n:
        x_ids, x_w = ids[indptr[rows]:indptr[rows + 1]], w[indptr[rows]:indptr[rows + 1]]
        m = x_ids.size
        elem = np.broadcast_to(x_ids, (k, m))
        coord = np.broadcast_to(np.arange(k, dtype=np.uint64)[:, None], (k, m))

        def u(stream):
            h = orc.hash64_array(elem, 0, 0, coord, 0, 0, stream)
            return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        r = -(np.log1p(-u(6)) + np.log1p(-u(7)))
        c = -(np.log1p(-u(8)) + np.log1p(-u(9)))
        beta = u(10)
        tick = np.floor(np.log(np.broadcast_to(x_w, (k, m))) / r + beta)
        ln_a = np.log(c) - r * (tick - beta) - r
        np.argmin(ln_a, axis=1)
        rows += 1
    cdt = time.perf_counter() - t0
    return {"row": "ICWS comparator", "metric": "sketches/sec", "value": n / (ms / 1e3),
            "unit": "sketches/sec", "ms_per_step": ms,
            "config": {"workload": "cfg3 rows", "sets": n, "nnz": 64, "k": k},
            "cpu_baseline": {"value": rows / cdt, "unit": "sketches/sec", "cores": 1,
                             "kind": "port",
                             "sample": f"first {rows} sets, numpy restatement, 1 thread"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--row", default="all", choices=["all", "bottomk", "lshindex", "dsk1", "icws"])
    args = ap.parse_args()
    import torch
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    rows = ["bottomk", "lshindex", "dsk1", "icws"] if args.row == "all" else [args.row]
    for r in rows:
        res = {"bottomk": row_bottomk, "lshindex": row_lshindex, "dsk1": row_dsk1,
               "icws": row_icws}[r](dev)
        for line in (res if isinstance(res, list) else [res]):
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
