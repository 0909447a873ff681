"""(L, K) LSH index over weighted sets with a GPU bulk path.

Mirrors LshIndex of the reference (ref/annindex.py:85-158): points live in
weight classes ||x||_1 in [2^c, 2^(c+1)); each point is normalised by 2^-c
and stored in L tables under the mix64 of its K smallest-rank darts per
table; a query probes every class its norm can share a similarity >= j1
with (probe_classes, ref/annindex.py:47-61), collects the points that share
a table key and scores them with exact weighted Jaccard, best first.

B200 layout: keys come from the K5 kernel (dsk_lsh_csr, normalisation
fused); the tables are one device array of (table id, key) -> point index
entries sorted once per batch of inserts, so a query batch is a pair of
device searchsorted calls; candidates are scored by the dsk_exact_jaccard
kernel on id-sorted copies of the sets.  Point ids are arbitrary hashables
kept on the host, like the reference's dict keys.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .api import (LshParams, ValidationError, WeightedSet, _device, _gather_rows, _lexsort_dev,
                  _ptr, _stream_ptr, _to_dev, lsh_batch, weight_class)

_CLASS_OFFSET = 1100  # weight classes lie in [-1075, 1024)


def probe_classes(l1: float, j1: float) -> list[int]:
    """Weight classes intersecting [j1*l1, l1/j1) (ref/annindex.py:47-61)."""
    lo = j1 * l1
    hi = l1 / j1
    c = weight_class(lo)
    out = []
    while math.ldexp(1.0, c) < hi:
        out.append(c)
        c += 1
    return out


def _sorted_rows(p: torch.Tensor, i: torch.Tensor, w: torch.Tensor):
    """Copy of a CSR batch with ids sorted ascending inside every row."""
    rows = torch.repeat_interleave(torch.arange(p.numel() - 1, device=p.device), p[1:] - p[:-1])
    flip = torch.tensor(-(2**63), dtype=torch.int64, device=p.device)
    order = _lexsort_dev([i ^ flip, rows])
    return p, i[order].contiguous(), w[order].contiguous()


class LshIndex:
    """Near-neighbour index over weighted sets (ref/annindex.py:85-158)."""

    def __init__(self, params: LshParams, hashes, debug: bool = False, device=None):
        self.params = params
        self.hashes = hashes
        self.device = _device(device)
        self._ids: list = []              # point index -> point id
        self._pos: dict = {}              # point id -> point index
        self._sets: list[WeightedSet] = []
        self._debug_keys = {} if debug else None
        # device state
        self._p = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._i = torch.zeros(0, dtype=torch.int64, device=self.device)
        self._w = torch.zeros(0, dtype=torch.float64, device=self.device)
        self._cls = torch.zeros(0, dtype=torch.int64, device=self.device)
        self._keys = torch.zeros((0, params.L), dtype=torch.int64, device=self.device)
        self._tables = None  # (unique keys, sorted composite codes, point index per code)

    def __len__(self) -> int:
        return len(self._ids)

    def __contains__(self, point_id) -> bool:
        return point_id in self._pos

    def point(self, point_id) -> WeightedSet:
        return self._sets[self._pos[point_id]]

    # ---------------------------------------------------------------- insert
    def insert(self, point_id, x: WeightedSet) -> None:
        """Index x under point_id in the weight class of its norm (ref/annindex.py:124-138)."""
        self.insert_many([point_id], [x])

    def insert_many(self, point_ids, sets) -> None:
        """Batch insert: classes, normalisation and keys for all sets in one
        kernel launch; the tables are rebuilt lazily at the next query."""
        point_ids = list(point_ids)
        sets = list(sets)
        if len(point_ids) != len(sets):
            raise ValueError("point_ids and sets differ in length")
        if not sets:
            return
        lens = np.fromiter((x.l0 for x in sets), dtype=np.int64, count=len(sets))
        new_ids = set(point_ids)
        if len(new_ids) != len(point_ids) or not new_ids.isdisjoint(self._pos.keys()):
            seen = set()
            for pid in point_ids:  # report the first offender, as insert() would
                if pid in self._pos or pid in seen:
                    raise ValidationError(f"duplicate point id {pid!r}")
                seen.add(pid)
        if (lens == 0).any():
            raise ValidationError("cannot index an empty set")
        dev = self.device
        indptr = np.zeros(lens.size + 1, dtype=np.int64)
        np.cumsum(lens, out=indptr[1:])
        ids = np.concatenate([x.ids for x in sets])
        w = np.concatenate([x.weights for x in sets])
        res = lsh_batch(indptr, ids, w, self.params, self.hashes, normalize=True, device=dev)
        # weight classes (ref/annindex.py:39-44): frexp exponent - 1 of each l1
        l1 = np.fromiter((x.l1 for x in sets), dtype=np.float64, count=len(sets))
        if not (l1 > 0).all():
            raise ValidationError("weight class requires a positive norm")
        cls = torch.from_numpy(np.frexp(l1)[1].astype(np.int64) - 1).to(dev)
        p_new, i_new, w_new = _sorted_rows(_to_dev(indptr, torch.int64, dev),
                                           _to_dev(ids, torch.int64, dev),
                                           _to_dev(w, torch.float64, dev))
        base = int(self._p[-1].item())
        self._p = torch.cat([self._p, p_new[1:] + base])
        self._i = torch.cat([self._i, i_new])
        self._w = torch.cat([self._w, w_new])
        self._cls = torch.cat([self._cls, cls])
        self._keys = torch.cat([self._keys, res.keys])
        first = len(self._ids)
        self._pos.update(zip(point_ids, range(first, first + len(point_ids))))
        self._ids.extend(point_ids)
        self._sets.extend(sets)
        if self._debug_keys is not None:
            keys = res.keys.cpu().numpy().view(np.uint64)
            for r, (pid, x) in enumerate(zip(point_ids, sets)):
                self._debug_keys[pid] = (weight_class(x.l1), keys[r])
        self._tables = None

    def bulk_load(self, path) -> list[int]:
        """Insert every set of a text file (ref/annindex.py:108-122)."""
        from .io import read_sets
        sets = read_sets(path)
        ids, next_id = [], len(self._ids)
        for _ in sets:
            while next_id in self._pos:
                next_id += 1
            ids.append(next_id)
            next_id += 1
        self.insert_many(ids, sets)
        return ids

    def _build_tables(self):
        L = self.params.L
        n = len(self._ids)
        dev = self.device
        flip = torch.tensor(-(2**63), dtype=torch.int64, device=dev)
        keyf = (self._keys ^ flip).reshape(-1)                       # unsigned order
        tid = ((self._cls + _CLASS_OFFSET).unsqueeze(1) * L +
               torch.arange(L, device=dev)).reshape(-1)
        pidx = torch.arange(n, device=dev).repeat_interleave(L)
        ukeys, inv = torch.unique(keyf, sorted=True, return_inverse=True)
        code = tid * ukeys.numel() + inv
        order = torch.argsort(code, stable=True)
        self._tables = (ukeys, code[order].contiguous(), pidx[order].contiguous())

    # ----------------------------------------------------------------- query
    def query(self, q: WeightedSet):
        """Candidates sharing a key with q in any probed class, scored with
        exact Jaccard on the stored vectors, best first (ref/annindex.py:140-158)."""
        return self.query_many([q])[0]

    def query_many(self, queries):
        queries = list(queries)
        for q in queries:
            if q.is_empty():
                raise ValidationError("cannot query with an empty set")
        out = [[] for _ in queries]
        if not queries or not self._ids:
            return out
        if self._tables is None:
            self._build_tables()
        ukeys, codes, pidx = self._tables
        L = self.params.L
        dev = self.device
        present = set(self._cls.unique().tolist())
        # one (query, probed class) row per probe, rescaled by 2^-c on the device
        pairs = [(qi, c) for qi, q in enumerate(queries) for c in probe_classes(q.l1, self.params.j1)
                 if c in present]
        if not pairs:
            return out
        lens = np.array([q.l0 for q in queries], dtype=np.int64)
        q_ptr = np.zeros(lens.size + 1, dtype=np.int64)
        np.cumsum(lens, out=q_ptr[1:])
        qp = _to_dev(q_ptr, torch.int64, dev)
        qi_ = _to_dev(np.concatenate([q.ids for q in queries]), torch.int64, dev)
        qw = _to_dev(np.concatenate([q.weights for q in queries]), torch.float64, dev)
        prow = torch.tensor([a for a, _ in pairs], dtype=torch.int64, device=dev)
        pcls = torch.tensor([c for _, c in pairs], dtype=torch.int64, device=dev)
        sp, si, sw = _gather_rows(qp, qi_, qw, prow)
        owner = torch.repeat_interleave(torch.arange(len(pairs), device=dev), sp[1:] - sp[:-1])
        sw = torch.ldexp(sw, -pcls[owner].to(torch.float64))  # scale_pow2(-c), exact
        res = lsh_batch(sp, si, sw, self.params, self.hashes, normalize=False, device=dev)
        # table lookups: code = (class, table) * |keys| + rank of the key
        flip = torch.tensor(-(2**63), dtype=torch.int64, device=dev)
        keyf = (res.keys ^ flip).reshape(-1)
        pos = torch.searchsorted(ukeys, keyf).clamp(max=ukeys.numel() - 1)
        hit = ukeys[pos] == keyf
        tid = ((pcls + _CLASS_OFFSET).unsqueeze(1) * L + torch.arange(L, device=dev)).reshape(-1)
        code = tid * ukeys.numel() + pos
        lo = torch.searchsorted(codes, code, right=False)
        hi = torch.searchsorted(codes, code, right=True)
        cnt = torch.where(hit, hi - lo, torch.zeros_like(lo))
        qrow = prow.repeat_interleave(L)
        total = int(cnt.sum().item())
        if total == 0:
            return out
        start = torch.repeat_interleave(lo, cnt, output_size=total)
        base = torch.repeat_interleave(torch.cumsum(cnt, 0) - cnt, cnt, output_size=total)
        cand = pidx[start + (torch.arange(total, device=dev) - base)]
        cq = torch.repeat_interleave(qrow, cnt, output_size=total)
        uniq = torch.unique(cq * len(self._ids) + cand)
        pq, pp = uniq // len(self._ids), uniq % len(self._ids)
        # exact Jaccard of each (query, candidate) on the unscaled vectors
        aq, ai, aw = _sorted_rows(qp, qi_, qw)
        scores = torch.empty(pq.numel(), dtype=torch.float64, device=dev)
        with torch.cuda.device(dev):
            _lib.check(_lib.load().dsk_exact_jaccard(
                _ptr(aq), _ptr(ai), _ptr(aw), _ptr(self._p), _ptr(self._i), _ptr(self._w),
                _ptr(pq), _ptr(pp), pq.numel(), _ptr(scores), _stream_ptr(dev)),
                "dsk_exact_jaccard")
        for a, b, sc in zip(pq.tolist(), pp.tolist(), scores.tolist()):
            out[a].append((self._ids[b], sc))
        for r in out:
            r.sort(key=lambda item: (-item[1], item[0]))
        return out

