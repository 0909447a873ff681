"""Python facade mirroring the reference's hot-path API on top of the C ABI.

Same names, argument meaning and error behaviour as the reference package
`dartsketch` (ref/ = /root/reference/pkg/src/dartsketch/):

  HashFamily(seed)                  ref/randomness.py:95-219
  WeightedSet, make_weighted_set    ref/core.py:23-100
  Dart, minhash_density             ref/core.py:123-156
  DartHasher(t, hashes)             ref/darthash.py:98-295 (darts, darts_below_rank, dart_batch)
  dart_minhash, MinHashSketch       ref/sketching.py:25-38, 115-123
  one_bit, OneBitSketch             ref/sketching.py:56-66, 164-167
  LshParams, weight_class, lsh_key  ref/annindex.py:24-82

plus batch entry points over CSR arrays (minhash_batch, lsh_batch,
darts_batch) that return device tensors.  Every computation runs in
libdsk_b200.so on the GPU; there is no CPU path.  uint64 values travel as
int64 bit patterns in torch tensors (view them as np.uint64 on the host).
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, constants
from .constants import ValidationError, minhash_density

DSK_OK, DSK_EMPTY, DSK_WEIGHT, DSK_DEPTH, DSK_AREAS, DSK_NOCONV, DSK_LIMIT = range(7)
DSK_OVERFLOW = 9
DSK_DUP = 10  # facade-level: a row repeats an element id (ref/core.py:42-43)
DSK_STATUS_TIE = 0x100

_STATUS_ERRORS = {
    DSK_EMPTY: (ValidationError, "cannot sketch an empty set"),
    DSK_WEIGHT: (ValidationError, "weights must be finite and strictly positive"),
    DSK_DEPTH: (ValidationError, "weights or rank limit outside the supported norm range"),
    DSK_AREAS: (ValidationError, "rank limit enumerates too many areas for this density"),
    DSK_NOCONV: (RuntimeError, "bucket filling did not converge; hash family is broken"),
    DSK_LIMIT: (ValidationError, "rank limit must be positive and finite"),
    7: (RuntimeError, "LSH hit buffer overflow (library limit)"),
    8: (RuntimeError, "set too large (reserved status)"),
    # 1 + t*x_i overflows to inf: math.floor(math.log2(inf)) raises in the
    # reference's depth computation (ref/darthash.py:154-156)
    DSK_OVERFLOW: (OverflowError, "cannot convert float infinity to integer"),
    DSK_DUP: (ValidationError, "duplicate element id"),
}


def _require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2005_11547_b200 runs on a CUDA device (B200, sm_100a); "
                           "there is no CPU path")


def _device(device) -> torch.device:
    _require_cuda()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ValueError("device must be a CUDA device")
    return torch.device("cuda", device.index if device.index is not None
                        else torch.cuda.current_device())


def _ptr(t) -> ctypes.c_void_p | None:
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_ptr(device: torch.device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _to_dev(a, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    """numpy / torch input -> contiguous device tensor (uint64 as int64 bits)."""
    if isinstance(a, torch.Tensor):
        t = a
        if t.dtype != dtype:
            if dtype == torch.int64 and t.dtype == torch.uint64:
                t = t.view(torch.int64)
            else:
                t = t.to(dtype)
        return t.to(device).contiguous()
    arr = np.asarray(a)
    if dtype == torch.int64 and arr.dtype == np.uint64:
        arr = arr.view(np.int64)
    elif dtype == torch.int64:
        arr = arr.astype(np.int64, copy=False)
    elif dtype == torch.float64:
        arr = arr.astype(np.float64, copy=False)
    arr = np.ascontiguousarray(arr)
    if not arr.flags.writeable:
        arr = arr.copy()
    return torch.from_numpy(arr).to(device)


def as_u64(t: torch.Tensor) -> np.ndarray:
    """Device int64 tensor of uint64 bit patterns -> host np.uint64 array."""
    return t.detach().cpu().numpy().view(np.uint64)


# ------------------------------------------------------------------ family


class HashFamily:
    """Tabulation-hash family seeded by a 64-bit value (ref/randomness.py:95-219).

    The tables are built on the host exactly like the reference and uploaded
    once per device into a libdsk_b200 context.  Immutable; shareable across
    threads (contexts are read-only after creation).
    """

    __slots__ = ("seed", "_tables", "poisson_cdf", "_ctx", "_cdf_dev", "_ctx_lock")

    def __init__(self, seed: int):
        seed = int(seed)
        self._tables = constants.hash_tables(seed)  # validates the 64-bit range
        self.seed = seed
        self.poisson_cdf = constants.poisson1_cdf()
        self._ctx = {}
        self._cdf_dev = {}
        self._ctx_lock = threading.Lock()

    def context(self, device=None) -> ctypes.c_void_p:
        """The libdsk_b200 context of this family on `device` (created once,
        thread-safely; the C calls themselves are reentrant)."""
        dev = _device(device)
        ctx = self._ctx.get(dev.index)
        if ctx is None:
            with self._ctx_lock:
                ctx = self._ctx.get(dev.index)
                if ctx is None:
                    lib = _lib.load()
                    out = ctypes.c_void_p()
                    thr = constants.log2_thresholds()
                    with torch.cuda.device(dev):
                        _lib.check(lib.dsk_ctx_create(dev.index, self._tables.ctypes.data,
                                                      self.poisson_cdf.ctypes.data,
                                                      thr.ctypes.data, ctypes.byref(out)),
                                   "dsk_ctx_create")
                    ctx = out
                    self._ctx[dev.index] = ctx
        return ctx

    def __del__(self):
        ctxs = getattr(self, "_ctx", None)
        if ctxs and _lib._lib is not None:
            for ctx in ctxs.values():
                try:
                    _lib._lib.dsk_ctx_destroy(ctx)
                except Exception:  # pragma: no cover - interpreter shutdown
                    pass
            ctxs.clear()

    # -- vectorized hashing (bit-identical to the reference's scalar path) ---
    def hash64_array(self, element, nu=0, rho=0, w=0, r=0, j=0, stream: int = 0,
                     device=None) -> np.ndarray:
        dev = _device(device)
        element = np.asarray(element, dtype=np.uint64)
        shape = element.shape
        cols = []
        for c, mask in ((element, None), (nu, 0xFF), (rho, 0xFF), (w, 0xFFFFFFFF),
                        (r, 0xFFFFFFFF), (j, 0xFFFF), (stream, 0xFFFF)):
            a = np.broadcast_to(np.asarray(c).astype(np.uint64), shape).ravel()
            cols.append(_to_dev(a, torch.int64, dev))
        out = torch.empty(int(np.prod(shape)), dtype=torch.int64, device=dev)
        lib = _lib.load()
        _lib.check(lib.dsk_hash64(self.context(dev), *[_ptr(c) for c in cols], out.numel(),
                                  _ptr(out), _stream_ptr(dev)), "dsk_hash64")
        return as_u64(out).reshape(shape)

    def hash64(self, element: int, nu: int = 0, rho: int = 0, w: int = 0, r: int = 0,
               j: int = 0, stream: int = 0) -> int:
        return int(self.hash64_array(np.uint64(int(element) & (2**64 - 1)), nu & 0xFF,
                                     rho & 0xFF, w & 0xFFFFFFFF, r & 0xFFFFFFFF, j & 0xFFFF,
                                     stream & 0xFFFF).reshape(()))

    def _uniform_dev(self, h: np.ndarray, dev) -> torch.Tensor:
        t = _to_dev(h.ravel(), torch.int64, dev)
        top = torch.bitwise_and(torch.bitwise_right_shift(t, 11), (1 << 53) - 1)
        return top.to(torch.float64) * (2.0 ** -53)  # exact: < 2^53

    def uniform_array(self, element, nu=0, rho=0, w=0, r=0, j=0, stream: int = 0) -> np.ndarray:
        dev = _device(None)
        h = self.hash64_array(element, nu, rho, w, r, j, stream, device=dev)
        return self._uniform_dev(h, dev).cpu().numpy().reshape(h.shape)

    def _unpack_key(self, key):
        fields = list(key) if not isinstance(key, (int, np.integer)) else [key]
        if len(fields) > 6:
            raise ValidationError("index tuples have at most 6 fields")
        fields += [0] * (6 - len(fields))
        return tuple(int(f) for f in fields)

    def uniform(self, key, stream: int) -> float:
        e, nu, rho, w, r, j = self._unpack_key(key)
        return float(self.uniform_array(np.uint64(e), nu, rho, w, r, j, stream).reshape(()))

    def poisson1_array(self, element, nu=0, rho=0, w=0, r=0) -> np.ndarray:
        dev = _device(None)
        h = self.hash64_array(element, nu, rho, w, r, 0, 3, device=dev)
        u = self._uniform_dev(h, dev)
        cdf = self._cdf_dev.get(dev.index)
        if cdf is None:
            cdf = torch.from_numpy(self.poisson_cdf).to(dev)
            self._cdf_dev[dev.index] = cdf
        return torch.searchsorted(cdf, u, right=True).cpu().numpy().reshape(h.shape)

    def poisson1(self, key) -> int:
        e, nu, rho, w, r, _ = self._unpack_key(key)
        return int(self.poisson1_array(np.uint64(e), nu, rho, w, r).reshape(()))

    def fingerprint_array(self, element, nu=0, rho=0, w=0, r=0, j=0) -> np.ndarray:
        return self.hash64_array(element, nu, rho, w, r, j, 4)

    def fingerprint(self, index) -> int:
        e, nu, rho, w, r, j = self._unpack_key(index)
        return self.hash64(e, nu, rho, w, r, j, 4)

    def bucket_array(self, fps, k: int) -> np.ndarray:
        if k < 1:
            raise ValidationError("bucket count must be positive")
        h = self.hash64_array(np.asarray(fps, dtype=np.uint64), stream=5)
        return (h % np.uint64(k)).astype(np.int64)

    def bucket(self, fp: int, k: int) -> int:
        return int(self.bucket_array(np.uint64(fp), k).reshape(()))

    def mix64(self, values) -> int:
        """Order-sensitive fold of a sequence (ref/randomness.py:160-166)."""
        v = np.asarray([int(x) & (2**64 - 1) for x in values], dtype=np.uint64)
        return int(self.mix64_rows(v.reshape(1, -1))[0])

    def mix64_rows(self, rows: np.ndarray, device=None) -> np.ndarray:
        dev = _device(device)
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        nseq, ln = rows.shape
        vin = _to_dev(rows.ravel(), torch.int64, dev)
        out = torch.zeros(nseq, dtype=torch.int64, device=dev)
        _lib.check(_lib.load().dsk_mix64(self.context(dev), _ptr(vin), nseq, ln, _ptr(out),
                                         _stream_ptr(dev)), "dsk_mix64")
        return as_u64(out)


# -------------------------------------------------------------- domain types


class WeightedSet:
    """Immutable sparse vector of strictly positive weights (ref/core.py:23-66)."""

    __slots__ = ("ids", "weights", "l1")

    def __init__(self, ids: np.ndarray, weights: np.ndarray, l1: float):
        self.ids = ids
        self.weights = weights
        self.l1 = l1

    @classmethod
    def from_arrays(cls, ids, weights) -> "WeightedSet":
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        weights = np.ascontiguousarray(weights, dtype=np.float64)
        if ids.shape != weights.shape or ids.ndim != 1:
            raise ValidationError("ids and weights must be parallel 1-d arrays")
        if weights.size and not (np.isfinite(weights).all() and (weights > 0).all()):
            raise ValidationError("weights must be finite and strictly positive")
        if np.unique(ids).size != ids.size:
            raise ValidationError("duplicate element id")
        return cls(ids, weights, float(np.sum(weights)))

    @property
    def l0(self) -> int:
        return int(self.ids.size)

    @property
    def entries(self):
        return list(zip(self.ids.tolist(), self.weights.tolist()))

    def is_empty(self) -> bool:
        return self.ids.size == 0

    def scale_pow2(self, exponent: int) -> "WeightedSet":
        weights = np.ldexp(self.weights, exponent)
        return WeightedSet(self.ids, weights, float(np.sum(weights)))

    def __len__(self) -> int:
        return self.l0

    def __repr__(self) -> str:
        return f"WeightedSet(l0={self.l0}, l1={self.l1!r})"


def make_weighted_set(pairs) -> WeightedSet:
    """Validate (id, weight) pairs; zero weights are dropped (ref/core.py:69-100)."""
    ids, weights = [], []
    for entry in pairs:
        try:
            element, weight = entry
        except (TypeError, ValueError):
            raise ValidationError(f"expected (id, weight) pair, got {entry!r}") from None
        element = int(element)
        weight = float(weight)
        if not 0 <= element <= 2**64 - 1:
            raise ValidationError(f"element id {element} outside 64-bit range")
        if math.isnan(weight) or math.isinf(weight):
            raise ValidationError(f"weight for id {element} is not finite")
        if weight < 0:
            raise ValidationError(f"negative weight {weight} for id {element}")
        if weight == 0.0:
            continue
        ids.append(element)
        weights.append(weight)
    if len(set(ids)) != len(ids):
        raise ValidationError("duplicate element id")
    w = np.asarray(weights, dtype=np.float64)
    return WeightedSet(np.asarray(ids, dtype=np.uint64), w, float(np.sum(w)) if weights else 0.0)


@dataclass(frozen=True)
class Dart:
    """One dart hitting a set (ref/core.py:123-147)."""

    element: int
    nu: int
    rho: int
    w: int
    r: int
    j: int
    weight: float
    rank: float
    fingerprint: int

    @property
    def index(self):
        return (self.element, self.nu, self.rho, self.w, self.r, self.j)


@dataclass(eq=False)
class MinHashSketch:
    values: np.ndarray
    k: int
    seed: int

    def __eq__(self, other):
        return (isinstance(other, MinHashSketch) and self.k == other.k
                and self.seed == other.seed and np.array_equal(self.values, other.values))

    def __len__(self) -> int:
        return self.k


@dataclass(eq=False)
class OneBitSketch:
    bits: np.ndarray
    k: int
    seed: int

    def __eq__(self, other):
        return (isinstance(other, OneBitSketch) and self.k == other.k
                and self.seed == other.seed and np.array_equal(self.bits, other.bits))

    def __len__(self) -> int:
        return self.k


@dataclass(frozen=True)
class LshParams:
    """L tables, K hashes per table, target similarity j1 (ref/annindex.py:24-36)."""

    L: int
    K: int
    j1: float = 0.5

    def __post_init__(self):
        if self.L < 1 or self.K < 1:
            raise ValidationError("L and K must be positive")
        if not 0.0 < self.j1 <= 1.0:
            raise ValidationError("j1 must lie in (0, 1]")


def weight_class(l1: float) -> int:
    """Exponent c with l1 in [2^c, 2^(c+1)) (ref/annindex.py:39-44)."""
    if not l1 > 0:
        raise ValidationError("weight class requires a positive norm")
    _, exponent = math.frexp(l1)
    return exponent - 1


# ------------------------------------------------------------ batch results


@dataclass
class MinhashBatch:
    values: torch.Tensor | None   # int64 [n, k]   (uint64 fingerprints)
    bits: torch.Tensor | None     # int64 [n, ceil(k/64)] packed one-bit words
    status: torch.Tensor          # int32 [n]
    phi: torch.Tensor             # int32 [n]     the reference's final phi step
    stats: torch.Tensor | None    # int32 [n, 4]  areas, candidate darts, hits, phi


@dataclass
class LshBatch:
    keys: torch.Tensor | None     # int64 [n, L]  mix64 of each table's K fingerprints
    fps: torch.Tensor | None      # int64 [n, L, K]
    status: torch.Tensor
    phi: torch.Tensor
    stats: torch.Tensor | None


def _csr_to_dev(indptr, ids, weights, dev):
    p = _to_dev(indptr, torch.int64, dev)
    i = _to_dev(ids, torch.int64, dev)
    w = _to_dev(weights, torch.float64, dev)
    return p, i, w


def raise_for_status(status: torch.Tensor, offset: int = 0, dup_rows=None) -> None:
    """Raise the reference's exception for the first failing row (row order).

    `dup_rows` (sorted row indices whose ids repeat, from `_dup_rows`) fail
    first on their row: the reference rejects them when the WeightedSet is
    built (ref/core.py:42-43), before anything is sketched."""
    st = status.cpu().numpy() & 0xFF
    bad = np.nonzero(st)[0]
    first_dup = int(dup_rows[0]) if dup_rows is not None and len(dup_rows) else None
    if first_dup is not None and (not bad.size or first_dup <= int(bad[0])):
        exc, msg = _STATUS_ERRORS[DSK_DUP]
        raise exc(f"set {first_dup + offset}: {msg}")
    if bad.size:
        row = int(bad[0])
        exc, msg = _STATUS_ERRORS.get(int(st[row]), (RuntimeError, f"status {int(st[row])}"))
        raise exc(f"set {row + offset}: {msg}")


def _dup_rows(p: torch.Tensor, i: torch.Tensor) -> np.ndarray:
    """Rows of a device CSR batch that repeat an element id (ascending).

    WeightedSet.from_arrays rejects them (ref/core.py:42-43); the batch
    entry points take raw CSR, so the facade checks on the device: one
    stable sort by id, one stable sort by row, adjacent equal (row, id)."""
    n = p.numel() - 1
    if i.numel() < 2 or n < 1:
        return np.zeros(0, dtype=np.int64)
    rows = torch.repeat_interleave(torch.arange(n, device=p.device), p[1:] - p[:-1])
    o = torch.sort(i, stable=True).indices
    o = o[torch.sort(rows[o], stable=True).indices]
    si, sr = i[o], rows[o]
    dup = (si[1:] == si[:-1]) & (sr[1:] == sr[:-1])
    return torch.unique(sr[1:][dup]).cpu().numpy()


HINT_DIRECT = 1 << 62  # DSK_HINT_DIRECT (include/dsk_b200.h)


def _shape_hint(indptr, p: torch.Tensor, i: torch.Tensor, weights=None,
                w: torch.Tensor | None = None) -> int:
    """Hints for dsk_minhash_csr_ex (results never depend on them).

    Team shape: the batch's nonzeros, or 0 (no hint) when at least half of
    ~4096 evenly spaced rows hold < 48 elements -- mostly-small batches
    (cfg5's Zipf sizes) run faster on single-warp teams whatever their mean.
    Direct-first (bit 62): at least 90 % of 256 evenly spaced rows have
    l1 > 2, so every band up to phi = 2 has rank depth 0 and the direct-only
    first launch serves nearly every set (cfg3's raw weights: 10-12 % faster;
    cfg2's normalised ones would all be handed back, so they do not get it).
    Host arrays are sampled on the host; device ones only for batches of
    >= 4096 rows (dsk_minhash_hints: one small launch + an 8-byte copy; this
    function then returns -1), smaller batches keep the mean-based hint (their
    shape follows the one-wave rule anyway)."""
    n = p.numel() - 1
    if n < 1:
        return 0
    m = min(n, 4096)
    md = min(n, 256)
    if isinstance(indptr, np.ndarray) and (weights is None or isinstance(weights, np.ndarray)):
        rows = np.arange(m, dtype=np.int64) * n // m
        small = int(np.count_nonzero((indptr[rows + 1] - indptr[rows]) < 48))
        direct = 0
        if weights is not None and n >= 4096:
            for r in (np.arange(md, dtype=np.int64) * n // md).tolist():
                direct += float(weights[indptr[r]:min(indptr[r + 1], indptr[r] + 4096)].sum()) > 2.0
    else:
        return -1  # device arrays: dsk_minhash_hints samples them (minhash_batch)
    hint = 0 if 2 * small >= m else i.numel()
    if n >= 4096 and 10 * direct >= 9 * md:
        hint |= HINT_DIRECT
    return hint


def _batch_hint(indptr, p, i, weights, w, hashes: "HashFamily", dev) -> int:
    """_shape_hint, with device arrays sampled by dsk_minhash_hints."""
    hint = _shape_hint(indptr, p, i, weights, w)
    if hint < 0:
        h = ctypes.c_int64(0)
        with torch.cuda.device(dev):
            _lib.check(_lib.load().dsk_minhash_hints(
                hashes.context(dev), _ptr(p), _ptr(w), p.numel() - 1, i.numel(), ctypes.byref(h),
                _stream_ptr(dev)), "dsk_minhash_hints")
        hint = h.value
    return hint


def minhash_batch(indptr, ids, weights, k: int, hashes: HashFamily, *, values: bool = True,
                  bits: bool = False, stats: bool = True, device=None,
                  check: bool = True) -> MinhashBatch:
    """dart_minhash for every row of a CSR batch, on the GPU."""
    if k < 1:
        raise ValidationError(f"k must be positive, got {k}")
    dev = _device(device)
    p, i, w = _csr_to_dev(indptr, ids, weights, dev)
    n = p.numel() - 1
    words = (k + 63) // 64
    out_v = torch.empty((n, k), dtype=torch.int64, device=dev) if values else None
    out_b = torch.empty((n, words), dtype=torch.int64, device=dev) if bits else None
    status = torch.empty(n, dtype=torch.int32, device=dev)
    phi = torch.empty(n, dtype=torch.int32, device=dev)
    st = torch.empty((n, 4), dtype=torch.int32, device=dev) if stats else None
    with torch.cuda.device(dev):
        hint = _batch_hint(indptr, p, i, weights, w, hashes, dev)
        _lib.check(_lib.load().dsk_minhash_csr_ex(
            hashes.context(dev), _ptr(p), _ptr(i), _ptr(w), n, int(k), hint, _ptr(out_v),
            _ptr(out_b), _ptr(status), _ptr(phi), _ptr(st), _stream_ptr(dev)), "dsk_minhash_csr")
    res = MinhashBatch(out_v, out_b, status, phi, st)
    if check:
        raise_for_status(status, dup_rows=_dup_rows(p, i))
        if bool(((status & DSK_STATUS_TIE) != 0).any()):
            _resolve_minhash_ties(res, p, i, w, k, hashes, dev)
    return res


def lsh_batch(indptr, ids, weights, params: LshParams, hashes: HashFamily, *,
              normalize: bool = False, keys: bool = True, fps: bool = False,
              stats: bool = True, device=None, check: bool = True) -> LshBatch:
    """lsh_key + per-table mix64 for every row of a CSR batch, on the GPU."""
    dev = _device(device)
    p, i, w = _csr_to_dev(indptr, ids, weights, dev)
    n = p.numel() - 1
    L, K = params.L, params.K
    out_k = torch.empty((n, L), dtype=torch.int64, device=dev) if keys else None
    out_f = torch.empty((n, L, K), dtype=torch.int64, device=dev) if fps else None
    status = torch.empty(n, dtype=torch.int32, device=dev)
    phi = torch.empty(n, dtype=torch.int32, device=dev)
    st = torch.empty((n, 4), dtype=torch.int32, device=dev) if stats else None
    # team-shape hint (results never depend on it): the largest row, looked
    # up (device arrays: one reduction + sync) only in the range of batch
    # sizes where the shape depends on it
    max_row = 0
    if 16384 <= n < 400000:
        max_row = int(np.diff(indptr).max()) if isinstance(indptr, np.ndarray) else \
            int((p[1:] - p[:-1]).max())
    with torch.cuda.device(dev):
        _lib.check(_lib.load().dsk_lsh_csr_ex(
            hashes.context(dev), _ptr(p), _ptr(i), _ptr(w), n, L, K, int(bool(normalize)),
            max_row, _ptr(out_k), _ptr(out_f), _ptr(status), _ptr(phi), _ptr(st),
            _stream_ptr(dev)), "dsk_lsh_csr")
    res = LshBatch(out_k, out_f, status, phi, st)
    if check:
        raise_for_status(status, dup_rows=_dup_rows(p, i))
        if bool(((status & DSK_STATUS_TIE) != 0).any()):
            _resolve_lsh_ties(res, p, i, w, params, hashes, dev, normalize)
    return res


def _resolve_lsh_ties(res: LshBatch, p, i, w, params: LshParams, hashes, dev,
                      normalize: bool) -> None:
    """Re-key the tables of sets whose darts had bit-identical ranks.

    The fast path orders a bucket's equal ranks by fingerprint; the
    reference orders them by index tuple (ref/annindex.py:77-81).  For the
    (astronomically rare) flagged sets, materialise the darts at phi* on the
    GPU, order each bucket by (rank, element, nu, rho, w, r, j), keep the K
    smallest and fold them with mix64 (ref/annindex.py:135).
    """
    tied = torch.nonzero((res.status & DSK_STATUS_TIE) != 0).flatten()
    if tied.numel() == 0:
        return
    L, K = params.L, params.K
    rows = tied.cpu().numpy()
    pp = p.cpu().numpy()
    sub_ptr = np.zeros(rows.size + 1, dtype=np.int64)
    np.cumsum(pp[rows + 1] - pp[rows], out=sub_ptr[1:])
    take = torch.cat([torch.arange(int(pp[r]), int(pp[r + 1]), device=dev) for r in rows])
    sub_ids = i[take]
    wh = w[take].cpu().numpy()
    l1 = np.empty(rows.size)
    for s in range(rows.size):
        seg = wh[sub_ptr[s]:sub_ptr[s + 1]]
        if normalize:  # LshIndex: scale_pow2(-weight_class(l1)), ref/annindex.py:130-131
            seg = np.ldexp(seg, -weight_class(float(np.sum(seg))))
            wh[sub_ptr[s]:sub_ptr[s + 1]] = seg
        l1[s] = float(np.sum(seg))
    limits = res.phi[tied].cpu().numpy().astype(np.float64) / l1
    offsets, status, cols = darts_batch(sub_ptr, sub_ids, wh, L * K, limits, hashes, device=dev)
    fp = cols["fingerprint"]
    h = _to_dev(hashes.hash64_array(as_u64(fp), stream=5, device=dev), torch.int64, dev)
    hi = torch.bitwise_and(torch.bitwise_right_shift(h, 32), 0xFFFFFFFF)
    lo = torch.bitwise_and(h, 0xFFFFFFFF)
    bucket = ((hi % L) * (1 << 32) + lo) % L
    owner = torch.repeat_interleave(torch.arange(rows.size, device=dev),
                                    offsets[1:] - offsets[:-1])
    flip = torch.tensor(-(2**63), dtype=torch.int64, device=dev)
    keys = [cols["j"].to(torch.int64), cols["r"].to(torch.int64) & 0xFFFFFFFF,
            cols["w"].to(torch.int64) & 0xFFFFFFFF, cols["rho"].to(torch.int64),
            cols["nu"].to(torch.int64), cols["element"] ^ flip, cols["rank"], bucket, owner]
    order = _lexsort_dev(keys)
    sb = owner[order] * L + bucket[order]
    first = torch.searchsorted(sb, sb, right=False)
    pos = torch.arange(order.numel(), device=dev) - first
    keep = pos < K
    tab = torch.zeros((rows.size * L, K), dtype=torch.int64, device=dev)
    tab[sb[keep], pos[keep]] = fp[order[keep]]
    if res.fps is not None:
        res.fps[tied] = tab.view(rows.size, L, K)
    if res.keys is not None:
        mixed = hashes.mix64_rows(as_u64(tab), device=dev)
        res.keys[tied] = _to_dev(mixed, torch.int64, dev).view(rows.size, L)
    res.status[tied] = res.status[tied] & 0xFF


DART_COLUMNS = (("element", torch.int64), ("nu", torch.int16), ("rho", torch.int16),
                ("w", torch.int32), ("r", torch.int32), ("j", torch.int16),
                ("weight", torch.float64), ("rank", torch.float64), ("fingerprint", torch.int64))


def darts_batch(indptr, ids, weights, t: int, rank_limit, hashes: HashFamily, *, device=None):
    """DartHasher(t).dart_batch for each row at its absolute rank limit.

    Returns (offsets int64[n+1], status int32[n], columns dict) on the device;
    the darts of row s are columns[...][offsets[s]:offsets[s+1]] (unordered).
    """
    t = int(t)
    if t < 1:
        raise ValidationError(f"density parameter t must be positive, got {t}")
    dev = _device(device)
    p, i, w = _csr_to_dev(indptr, ids, weights, dev)
    n = p.numel() - 1
    lim = _to_dev(np.broadcast_to(np.asarray(rank_limit, dtype=np.float64), (n,)).copy()
                  if not isinstance(rank_limit, torch.Tensor) else rank_limit, torch.float64, dev)
    counts = torch.zeros(n, dtype=torch.int64, device=dev)
    status = torch.zeros(n, dtype=torch.int32, device=dev)
    lib = _lib.load()
    ctx = hashes.context(dev)
    nulls = [None] * 9
    with torch.cuda.device(dev):
        _lib.check(lib.dsk_darts_csr(ctx, _ptr(p), _ptr(i), _ptr(w), n, t, _ptr(lim), None, 0,
                                     _ptr(counts), _ptr(status), *nulls, _stream_ptr(dev)),
                   "dsk_darts_csr(count)")
        offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        torch.cumsum(counts, 0, out=offsets[1:])
        total = int(offsets[-1].item())
        cols = {name: torch.zeros(max(total, 1), dtype=dt, device=dev) for name, dt in DART_COLUMNS}
        if total:
            _lib.check(lib.dsk_darts_csr(ctx, _ptr(p), _ptr(i), _ptr(w), n, t, _ptr(lim),
                                         _ptr(offsets), total, _ptr(counts), _ptr(status),
                                         *[_ptr(cols[name]) for name, _ in DART_COLUMNS],
                                         _stream_ptr(dev)), "dsk_darts_csr(fill)")
    cols = {k2: v[:total] for k2, v in cols.items()}
    return offsets, status, cols


def _resolve_minhash_ties(res: MinhashBatch, p, i, w, k, hashes, dev) -> None:
    """Re-resolve slots of sets whose darts had bit-identical ranks.

    The fast path orders equal ranks by fingerprint; the reference orders
    them by index tuple (ref/sketching.py:93-99).  For the (astronomically
    rare) flagged sets, materialise the darts at the final step on the GPU
    and take the per-bucket minimum by (rank, element, nu, rho, w, r, j).
    """
    tied = torch.nonzero((res.status & DSK_STATUS_TIE) != 0).flatten()
    if tied.numel() == 0:
        return
    rows = tied.cpu().numpy()
    pp = p.cpu().numpy()
    sub_ptr = np.zeros(rows.size + 1, dtype=np.int64)
    np.cumsum(pp[rows + 1] - pp[rows], out=sub_ptr[1:])
    take = torch.cat([torch.arange(int(pp[r]), int(pp[r + 1]), device=dev) for r in rows])
    sub_ids, sub_w = i[take], w[take]
    # final limit phi*/l1 per set: l1 = np.sum of the row (host numpy restates the reference)
    l1 = np.array([float(np.sum(sub_w[sub_ptr[s]:sub_ptr[s + 1]].cpu().numpy()))
                   for s in range(rows.size)])
    phis = res.phi[tied].cpu().numpy().astype(np.float64)
    limits = phis / l1
    offsets, status, cols = darts_batch(sub_ptr, sub_ids, sub_w, minhash_density(k), limits,
                                        hashes, device=dev)
    fp = cols["fingerprint"]
    h = _to_dev(hashes.hash64_array(as_u64(fp), stream=5, device=dev), torch.int64, dev)
    hi = torch.bitwise_and(torch.bitwise_right_shift(h, 32), 0xFFFFFFFF)
    lo = torch.bitwise_and(h, 0xFFFFFFFF)
    bucket = ((hi % k) * (1 << 32) + lo) % k
    owner = torch.repeat_interleave(torch.arange(rows.size, device=dev),
                                    offsets[1:] - offsets[:-1])
    flip = torch.tensor(-(2**63), dtype=torch.int64, device=dev)
    keys = [cols["j"].to(torch.int64), cols["r"].to(torch.int64) & 0xFFFFFFFF,
            cols["w"].to(torch.int64) & 0xFFFFFFFF, cols["rho"].to(torch.int64),
            cols["nu"].to(torch.int64), cols["element"] ^ flip, cols["rank"], bucket, owner]
    order = torch.arange(fp.numel(), device=dev)
    for key in keys:  # least significant first, stable: np.lexsort on the GPU
        order = order[torch.sort(key[order], stable=True).indices]
    sb = (owner[order] * k + bucket[order])
    first = torch.ones_like(sb, dtype=torch.bool)
    first[1:] = sb[1:] != sb[:-1]
    sel = order[first]
    # every bucket of a tied row is non-empty at phi*, so `sel` holds all k
    # minima of those rows: rebuild them whole (values and/or packed bits)
    fixed = torch.zeros((rows.size, k), dtype=torch.int64, device=dev)
    fixed[owner[sel], bucket[sel]] = fp[sel]
    if res.values is not None:
        res.values[tied] = fixed
    if res.bits is not None:
        words = res.bits.shape[1]
        packed = torch.zeros((rows.size, words), dtype=torch.int64, device=dev)
        _lib.check(_lib.load().dsk_pack_onebit(_ptr(fixed), rows.size, k, _ptr(packed),
                                               _stream_ptr(dev)), "dsk_pack_onebit")
        res.bits[tied] = packed
    res.status[tied] = res.status[tied] & 0xFF


# ------------------------------------------------------------- bottom-k


def l1_batch(indptr, weights, *, device=None) -> torch.Tensor:
    """float(np.sum(weights)) per CSR row (ref/core.py:44), on the GPU."""
    dev = _device(device)
    p = _to_dev(indptr, torch.int64, dev)
    w = _to_dev(weights, torch.float64, dev)
    out = torch.empty(p.numel() - 1, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().dsk_l1_csr(_ptr(p), _ptr(w), out.numel(), _ptr(out),
                                          _stream_ptr(dev)), "dsk_l1_csr")
    return out


def _gather_rows(p: torch.Tensor, i: torch.Tensor, w: torch.Tensor, rows: torch.Tensor):
    """Sub-CSR of the given rows, built on the device."""
    lengths = p[rows + 1] - p[rows]
    sub_p = torch.zeros(rows.numel() + 1, dtype=torch.int64, device=p.device)
    torch.cumsum(lengths, 0, out=sub_p[1:])
    total = int(sub_p[-1].item())
    start = torch.repeat_interleave(p[rows], lengths, output_size=total)
    base = torch.repeat_interleave(sub_p[:-1], lengths, output_size=total)
    take = start + (torch.arange(total, device=p.device) - base)
    return sub_p, i[take], w[take]


def _lexsort_dev(keys):
    """np.lexsort on the device: stable sorts, least significant key first."""
    order = torch.arange(keys[0].numel(), device=keys[0].device)
    for key in keys:
        order = order[torch.sort(key[order], stable=True).indices]
    return order


@dataclass
class BottomKBatch:
    columns: dict                 # name -> tensor [n, k] (DartBatch columns, rank order)
    status: torch.Tensor          # int32 [n]
    phi: torch.Tensor             # int32 [n]


def _bottom_k_composed(p, i, w, k: int, hashes: HashFamily, dev, check: bool) -> BottomKBatch:
    """bottom_k composed from the darts kernel (K6) and a device lexsort per
    phi step; the fallback of the fused kernel (sets whose darts outgrow its
    buffer, or k above its range)."""
    n = p.numel() - 1
    l1 = l1_batch(p, w, device=dev)
    cols = {name: torch.zeros((n, k), dtype=dt, device=dev) for name, dt in DART_COLUMNS}
    status = torch.zeros(n, dtype=torch.int32, device=dev)
    phis = torch.zeros(n, dtype=torch.int32, device=dev)
    empty = (p[1:] - p[:-1]) == 0
    status[empty] = DSK_EMPTY
    pending = torch.nonzero(~empty).flatten()
    flip = torch.tensor(-(2**63), dtype=torch.int64, device=dev)
    for phi in range(1, 65):  # ref/sketching.py:150
        if pending.numel() == 0:
            break
        sp, si, sw = _gather_rows(p, i, w, pending)
        limits = float(phi) / l1[pending]
        offsets, st, dc = darts_batch(sp, si, sw, k, limits, hashes, device=dev)
        bad = st != 0
        if bool(bad.any()):
            status[pending[bad]] = st[bad]
        counts = offsets[1:] - offsets[:-1]
        done = (counts >= k) & ~bad
        if bool(done.any()):
            owner = torch.repeat_interleave(torch.arange(pending.numel(), device=dev), counts)
            sel_dart = done[owner]
            idx = torch.nonzero(sel_dart).flatten()
            o = owner[idx]
            keys = [dc["j"][idx].to(torch.int64), dc["r"][idx].to(torch.int64) & 0xFFFFFFFF,
                    dc["w"][idx].to(torch.int64) & 0xFFFFFFFF, dc["rho"][idx].to(torch.int64),
                    dc["nu"][idx].to(torch.int64), dc["element"][idx] ^ flip, dc["rank"][idx], o]
            order = idx[_lexsort_dev(keys)]
            oo = owner[order]
            first = torch.searchsorted(oo, oo, right=False)
            pos = torch.arange(order.numel(), device=dev) - first
            keep = pos < k
            rows_out = pending[oo[keep]]
            for name, _ in DART_COLUMNS:
                cols[name][rows_out, pos[keep]] = dc[name][order[keep]]
            phis[pending[done]] = phi
        pending = pending[~done & ~bad]
    if pending.numel():
        status[pending] = DSK_NOCONV
    res = BottomKBatch(cols, status, phis)
    if check:
        raise_for_status(status)
    return res


_BOTTOMK_FUSED_MAX_K = 256  # counting-rank selection cost grows with k^2


def bottom_k_batch(indptr, ids, weights, k: int, hashes: HashFamily, *, device=None,
                   check: bool = True) -> BottomKBatch:
    """bottom_k for every CSR row (ref/sketching.py:146-156): density t = k;
    at the first phi step with >= k darts, the k smallest by (rank, index).

    k <= 256: one fused kernel (dsk_bottomk_csr); rows it cannot hold in its
    buffer, and larger k, go through the composed darts + lexsort path."""
    k = int(k)
    if k < 1:
        raise ValidationError(f"k must be positive, got {k}")
    dev = _device(device)
    p, i, w = _csr_to_dev(indptr, ids, weights, dev)
    n = p.numel() - 1
    if k > _BOTTOMK_FUSED_MAX_K:
        return _bottom_k_composed(p, i, w, k, hashes, dev, check)
    cols = {name: torch.zeros((n, k), dtype=dt, device=dev) for name, dt in DART_COLUMNS}
    status = torch.zeros(n, dtype=torch.int32, device=dev)
    phis = torch.zeros(n, dtype=torch.int32, device=dev)
    order = [cols[name] for name, _ in DART_COLUMNS]
    with torch.cuda.device(dev):
        _lib.check(_lib.load().dsk_bottomk_csr(
            hashes.context(dev), _ptr(p), _ptr(i), _ptr(w), n, k, *[_ptr(c) for c in order],
            _ptr(status), _ptr(phis), _stream_ptr(dev)), "dsk_bottomk_csr")
    spill = torch.nonzero(status == 7).flatten()  # DSK_SCRATCH: recompute those rows
    if spill.numel():
        sp, si, sw = _gather_rows(p, i, w, spill)
        sub = _bottom_k_composed(sp, si, sw, k, hashes, dev, False)
        for name, _ in DART_COLUMNS:
            cols[name][spill] = sub.columns[name]
        status[spill] = sub.status
        phis[spill] = sub.phi
    res = BottomKBatch(cols, status, phis)
    if check:
        raise_for_status(status, dup_rows=_dup_rows(p, i))
    return res


@dataclass(eq=False)
class BottomKSketch:
    """The k smallest-rank darts hitting a set, ascending (ref/sketching.py:40-53)."""

    darts: list
    k: int
    seed: int

    @property
    def fingerprints(self) -> np.ndarray:
        return np.asarray([d.fingerprint for d in self.darts], dtype=np.uint64)

    def __eq__(self, other):
        return (isinstance(other, BottomKSketch) and self.k == other.k
                and self.seed == other.seed and self.darts == other.darts)

    def __len__(self) -> int:
        return self.k


@dataclass(frozen=True)
class BottomKFingerprints:
    """Deserialized bottom-k record (ref/sketching.py:71-77)."""

    values: np.ndarray = dataclasses.field(compare=False)
    k: int = 0
    seed: int = 0


def bottom_k(x: WeightedSet, k: int, hashes: HashFamily) -> BottomKSketch:
    """The first k darts hitting x, in ascending rank order (ref/sketching.py:146-156)."""
    if x.is_empty():
        raise ValidationError("cannot sketch an empty set")
    if k < 1:
        raise ValidationError(f"k must be positive, got {k}")
    res = bottom_k_batch(*_single_csr(x), k, hashes)
    h = {name: v[0].cpu().numpy() for name, v in res.columns.items()}
    batch = DartBatch(h["element"].view(np.uint64), h["nu"].view(np.uint16),
                      h["rho"].view(np.uint16), h["w"].view(np.uint32), h["r"].view(np.uint32),
                      h["j"].view(np.uint16), h["weight"], h["rank"],
                      h["fingerprint"].view(np.uint64))
    return BottomKSketch(batch.to_darts(), k, hashes.seed)


# ---------------------------------------------------------- DSK1 records

SKETCH_MAGIC = b"DSK1"
SKETCH_VERSION = 1
KIND_MINHASH, KIND_ONEBIT, KIND_BOTTOMK = 1, 2, 3
_HEADER_BYTES = 20  # struct "<4sBBHIQ", ref/sketching.py:221


def dump_sketches(payload: torch.Tensor, kind: int, k: int, seed: int) -> bytes:
    """DSK1 records for a batch, byte-identical to b"".join(dump_sketch(s) ...)
    (ref/sketching.py:224-231), written on the GPU.

    payload: device int64 tensor [n, k] of uint64 values (minhash, bottom-k
    fingerprints) or [n, ceil(k/64)] packed one-bit words (kind 2)."""
    dev = payload.device
    n = payload.shape[0]
    pbytes = (k + 7) // 8 if kind == KIND_ONEBIT else 8 * k
    out = torch.empty(n * (_HEADER_BYTES + pbytes), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().dsk_dsk1_records(int(kind), int(k), int(seed) & (2**64 - 1),
                                                _ptr(payload.contiguous()), n, _ptr(out),
                                                _stream_ptr(dev)), "dsk_dsk1_records")
    host = torch.empty(out.numel(), dtype=torch.uint8, pin_memory=True)
    host.copy_(out, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    return host.numpy().tobytes()


def dump_sketch(sketch) -> bytes:
    """Serialize one sketch (ref/sketching.py:224-231)."""
    dev = _device(None)
    if isinstance(sketch, MinHashSketch):
        v = _to_dev(np.asarray(sketch.values, dtype=np.uint64), torch.int64, dev).view(1, -1)
        return dump_sketches(v, KIND_MINHASH, sketch.k, sketch.seed)
    if isinstance(sketch, OneBitSketch):
        bits = np.asarray(sketch.bits, dtype=np.uint8)
        words = (sketch.k + 63) // 64
        packed = np.zeros(words * 8, dtype=np.uint8)
        pb = np.packbits(bits, bitorder="little")
        packed[:pb.size] = pb
        v = _to_dev(packed.view("<u8"), torch.int64, dev).view(1, -1)
        return dump_sketches(v, KIND_ONEBIT, sketch.k, sketch.seed)
    if isinstance(sketch, (BottomKSketch, BottomKFingerprints)):
        vals = sketch.fingerprints if isinstance(sketch, BottomKSketch) else sketch.values
        v = _to_dev(np.asarray(vals, dtype=np.uint64), torch.int64, dev).view(1, -1)
        return dump_sketches(v, KIND_BOTTOMK, sketch.k, sketch.seed)
    raise ValidationError(f"cannot serialize object of type {type(sketch).__name__}")


def iter_sketches(data: bytes):
    """Parse concatenated DSK1 records (ref/sketching.py:234-281)."""
    import struct
    hdr = struct.Struct("<4sBBHIQ")
    off = 0
    while off < len(data):
        if len(data) - off < hdr.size:
            raise ValidationError("truncated sketch record")
        magic, version, kind, _, k, seed = hdr.unpack_from(data, off)
        if magic != SKETCH_MAGIC:
            raise ValidationError(f"bad sketch magic {magic!r}")
        if version != SKETCH_VERSION:
            raise ValidationError(f"unsupported sketch version {version}")
        off += hdr.size
        size = (k + 7) // 8 if kind == KIND_ONEBIT else 8 * k
        if len(data) - off < size:
            raise ValidationError("truncated sketch payload")
        payload = data[off:off + size]
        off += size
        if kind == KIND_MINHASH:
            yield MinHashSketch(np.frombuffer(payload, dtype="<u8").astype(np.uint64), k, seed)
        elif kind == KIND_ONEBIT:
            bits = np.unpackbits(np.frombuffer(payload, dtype=np.uint8), count=k,
                                 bitorder="little")
            yield OneBitSketch(bits, k, seed)
        elif kind == KIND_BOTTOMK:
            yield BottomKFingerprints(np.frombuffer(payload, dtype="<u8").astype(np.uint64), k,
                                      seed)
        else:
            raise ValidationError(f"unknown sketch kind {kind}")


def load_sketch(data: bytes, offset: int = 0):
    return next(iter_sketches(data[offset:]))


# --------------------------------------------------------- single-set API


def _single_csr(x: WeightedSet):
    return np.array([0, x.l0], dtype=np.int64), x.ids, x.weights


def dart_minhash(x: WeightedSet, k: int, hashes: HashFamily) -> MinHashSketch:
    """k independent weighted minhash values of x (ref/sketching.py:115-123)."""
    if x.is_empty():
        raise ValidationError("cannot sketch an empty set")
    if k < 1:
        raise ValidationError(f"k must be positive, got {k}")
    res = minhash_batch(*_single_csr(x), k, hashes, stats=False)
    return MinHashSketch(as_u64(res.values[0]).copy(), k, hashes.seed)


def one_bit(sketch: MinHashSketch) -> OneBitSketch:
    """Lowest bit of each minhash value (ref/sketching.py:164-167), on the GPU."""
    dev = _device(None)
    v = _to_dev(sketch.values, torch.int64, dev)
    bits = torch.bitwise_and(v, 1).to(torch.uint8).cpu().numpy()
    return OneBitSketch(bits, sketch.k, sketch.seed)


def lsh_key(x: WeightedSet, params: LshParams, hashes: HashFamily):
    """L tuples of the K smallest-rank fingerprints per table (ref/annindex.py:64-82)."""
    if x.is_empty():
        raise ValidationError("cannot key an empty set")
    res = lsh_batch(*_single_csr(x), params, hashes, keys=False, fps=True, stats=False)
    fps = as_u64(res.fps[0])
    return [tuple(int(v) for v in row) for row in fps]


def exact_jaccard(x: WeightedSet, y: WeightedSet, *, device=None) -> float:
    """Weighted Jaccard similarity sum(min) / sum(max) (ref/core.py:103-120),
    computed by the dsk_exact_jaccard kernel: both rows merged in ascending id
    order with sequential fp64 sums, as the reference's loop over
    sorted(union) does.  Raises ValidationError for two empty sets."""
    if x.is_empty() and y.is_empty():
        raise ValidationError("Jaccard similarity is undefined for two empty sets")
    dev = _device(device)
    ox, oy = np.argsort(x.ids, kind="stable"), np.argsort(y.ids, kind="stable")
    indptr = np.array([0, x.ids.size, x.ids.size + y.ids.size], dtype=np.int64)
    ids = np.concatenate([x.ids[ox], y.ids[oy]]).astype(np.uint64)
    ws = np.concatenate([x.weights[ox], y.weights[oy]]).astype(np.float64)
    p, i, w = _csr_to_dev(indptr, ids, ws, dev)
    pa = torch.zeros(1, dtype=torch.int64, device=dev)
    pb = torch.ones(1, dtype=torch.int64, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().dsk_exact_jaccard(_ptr(p), _ptr(i), _ptr(w), _ptr(p), _ptr(i),
                                                 _ptr(w), _ptr(pa), _ptr(pb), 1, _ptr(out),
                                                 _stream_ptr(dev)), "dsk_exact_jaccard")
    return float(out.item())


class DartBatch:
    """Column-oriented darts (ref/darthash.py:39-77)."""

    __slots__ = ("element", "nu", "rho", "w", "r", "j", "weight", "rank", "fingerprint")

    def __init__(self, element, nu, rho, w, r, j, weight, rank, fingerprint):
        self.element, self.nu, self.rho, self.w, self.r, self.j = element, nu, rho, w, r, j
        self.weight, self.rank, self.fingerprint = weight, rank, fingerprint

    @property
    def size(self) -> int:
        return int(self.element.size)

    @classmethod
    def empty(cls) -> "DartBatch":
        """A batch of no darts with the reference's column dtypes (ref/darthash.py:59-64)."""
        return cls(np.empty(0, np.uint64), np.empty(0, np.uint16), np.empty(0, np.uint16),
                   np.empty(0, np.uint32), np.empty(0, np.uint32), np.empty(0, np.uint16),
                   np.empty(0, np.float64), np.empty(0, np.float64), np.empty(0, np.uint64))

    def take(self, indices) -> "DartBatch":
        """The rows at `indices`, every column (ref/darthash.py:66-67)."""
        return DartBatch(*(getattr(self, name)[indices] for name in self.__slots__))

    def index_sort_keys(self):
        return (self.j, self.r, self.w, self.rho, self.nu, self.element)

    def to_darts(self):
        rows = zip(self.element.tolist(), self.nu.tolist(), self.rho.tolist(), self.w.tolist(),
                   self.r.tolist(), self.j.tolist(), self.weight.tolist(), self.rank.tolist(),
                   self.fingerprint.tolist())
        return [Dart(*row) for row in rows]


class DartHasher:
    """Enumerates darts at a fixed density t (ref/darthash.py:98-139), on the GPU."""

    __slots__ = ("t", "hashes")

    def __init__(self, t: int, hashes: HashFamily):
        t = int(t)
        if t < 1:
            raise ValidationError(f"density parameter t must be positive, got {t}")
        self.t = t
        self.hashes = hashes

    def darts(self, x: WeightedSet, phi: float):
        phi = float(phi)
        if not phi > 0 or math.isinf(phi):
            raise ValidationError(f"phi must be positive and finite, got {phi}")
        if x.is_empty():
            raise ValidationError("cannot throw darts at an empty set")
        return self.dart_batch(x, phi / x.l1).to_darts()

    def darts_below_rank(self, x: WeightedSet, rank_limit: float):
        if x.is_empty():
            raise ValidationError("cannot throw darts at an empty set")
        if not rank_limit > 0 or math.isinf(rank_limit):
            raise ValidationError(f"rank limit must be positive and finite, got {rank_limit}")
        return self.dart_batch(x, float(rank_limit)).to_darts()

    def dart_batch(self, x: WeightedSet, rank_limit: float) -> DartBatch:
        if x.is_empty():
            raise ValidationError("cannot throw darts at an empty set")
        if not rank_limit > 0 or math.isinf(rank_limit):
            raise ValidationError(f"rank limit must be positive and finite, got {rank_limit}")
        offsets, status, cols = darts_batch(*_single_csr(x), self.t, float(rank_limit),
                                            self.hashes)
        raise_for_status(status)
        h = {name: v.cpu().numpy() for name, v in cols.items()}
        return DartBatch(h["element"].view(np.uint64), h["nu"].view(np.uint16),
                         h["rho"].view(np.uint16), h["w"].view(np.uint32),
                         h["r"].view(np.uint32), h["j"].view(np.uint16), h["weight"],
                         h["rank"], h["fingerprint"].view(np.uint64))


__all__ = [
    "HashFamily", "WeightedSet", "make_weighted_set", "Dart", "DartBatch", "DartHasher",
    "MinHashSketch", "OneBitSketch", "LshParams", "weight_class", "minhash_density",
    "dart_minhash", "one_bit", "lsh_key", "minhash_batch", "lsh_batch", "darts_batch",
    "MinhashBatch", "LshBatch", "ValidationError", "raise_for_status", "as_u64",
    "DSK_STATUS_TIE", "l1_batch", "bottom_k_batch", "BottomKBatch", "BottomKSketch",
    "BottomKFingerprints", "bottom_k", "dump_sketches", "dump_sketch", "iter_sketches",
    "load_sketch", "exact_jaccard",
]
_ = dataclasses


# ------------------------------------------------- ICWS comparator (f4)


@dataclass(frozen=True)
class IcwsHashValue:
    """A consistent weighted sample: element id plus quantised log-weight tick
    (ref/baselines.py:75-81)."""

    element: int
    tick: int


@dataclass
class IcwsBatch:
    element: torch.Tensor  # int64 [n, k] (uint64 ids)
    tick: torch.Tensor     # int64 [n, k]
    status: torch.Tensor   # int32 [n]


def icws_batch(indptr, ids, weights, k: int, hashes: HashFamily, *, device=None,
               check: bool = True) -> IcwsBatch:
    """ICWS samples (ref/baselines.py:84-161) for every CSR row, on the GPU.

    A comparator, not DartMinHash: log / log1p are CUDA's, so a sample may
    differ from the host reference's where candidates tie to within an ulp
    (none in the tested fixtures)."""
    k = int(k)
    if k < 1:
        raise ValidationError(f"k must be positive, got {k}")
    dev = _device(device)
    p, i, w = _csr_to_dev(indptr, ids, weights, dev)
    n = p.numel() - 1
    el = torch.zeros((n, k), dtype=torch.int64, device=dev)
    tk = torch.zeros((n, k), dtype=torch.int64, device=dev)
    status = torch.zeros(n, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().dsk_icws_csr(hashes.context(dev), _ptr(p), _ptr(i), _ptr(w), n, k,
                                            _ptr(el), _ptr(tk), _ptr(status), _stream_ptr(dev)),
                   "dsk_icws_csr")
    res = IcwsBatch(el, tk, status)
    if check:
        raise_for_status(status, dup_rows=_dup_rows(p, i))
    return res


class IcwsSketcher:
    """Ioffe consistent weighted sampling with HashFamily randomness
    (ref/baselines.py:84-136); `fast` is accepted for API parity (the device
    computes log(x) once per element either way; outputs are identical)."""

    __slots__ = ("k", "hashes", "fast")

    def __init__(self, k: int, hashes: HashFamily, fast: bool = False):
        if k < 1:
            raise ValidationError(f"k must be positive, got {k}")
        self.k = k
        self.hashes = hashes
        self.fast = fast

    @property
    def seed(self) -> int:
        return self.hashes.seed

    def minhash(self, x: WeightedSet) -> list:
        if x.is_empty():
            raise ValidationError("cannot sketch an empty set")
        res = icws_batch(*_single_csr(x), self.k, self.hashes)
        el = as_u64(res.element[0])
        tk = res.tick[0].cpu().numpy()
        return [IcwsHashValue(int(e), int(t)) for e, t in zip(el, tk)]


def icws_minhash(x: WeightedSet, k: int, hashes: HashFamily, fast: bool = False) -> list:
    """k consistent weighted samples of x (ref/baselines.py:139-142)."""
    return IcwsSketcher(k, hashes, fast=fast).minhash(x)


def icws_estimate_jaccard(a: list, b: list) -> float:
    """Fraction of coordinates whose samples collide (ref/baselines.py:145-149)."""
    if len(a) != len(b):
        raise ValidationError("sketch lengths differ")
    return sum(u == v for u, v in zip(a, b)) / len(a)


def icws_fingerprints(values: list, hashes: HashFamily) -> np.ndarray:
    """64-bit fingerprints of ICWS samples (ref/baselines.py:152-161), on the GPU:
    hash64(element, w = tick low 32 bits, r = tick high 32 bits, stream 11)."""
    el = np.array([v.element & (2**64 - 1) for v in values], dtype=np.uint64)
    tk = np.array([v.tick & (2**64 - 1) for v in values], dtype=np.uint64)
    return hashes.hash64_array(el, w=tk & np.uint64(0xFFFFFFFF), r=tk >> np.uint64(32),
                               stream=11)
