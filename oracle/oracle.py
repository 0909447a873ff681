"""ctypes wrapper around the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY.  The oracle restates the reference package
`dartsketch` (ref/ = /root/reference/pkg/src/dartsketch/) in C; see
oracle/dsk_oracle.c for the per-function file:line citations.  It is the
parity checker for the CUDA path and the CPU baseline of bench.py; the
product package never imports it.

Pinned by tests/test_oracle.py against golden vectors the reference itself
produced (tests/golden/make_golden.py) and the reference's own known answers
(the hash golden 317886004245365293, minhash_density values).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

STATUS_NAMES = {0: "ok", 1: "empty", 2: "weight", 3: "depth", 4: "areas",
                5: "noconv", 6: "limit", 7: "badarg", 8: "nomem", 9: "overflow"}

DART_DTYPE = np.dtype([
    ("element", "<u8"), ("nu", "<u2"), ("rho", "<u2"), ("w", "<u4"), ("r", "<u4"),
    ("j", "<u2"), ("pad", "<u2"), ("weight", "<f8"), ("rank", "<f8"), ("fingerprint", "<u8"),
])


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc only)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "dsk_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE, "-B" if force else "all"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        P = ctypes.c_void_p
        L.or_hash64.restype = ctypes.c_uint64
        L.or_hash64.argtypes = [P] + [ctypes.c_uint64] * 7
        L.or_finalize.restype = ctypes.c_uint64
        L.or_finalize.argtypes = [ctypes.c_uint64]
        L.or_poisson1_cdf.argtypes = [P]
        L.or_mix64.restype = ctypes.c_uint64
        L.or_mix64.argtypes = [P, P, ctypes.c_int64]
        L.or_pairwise_sum.restype = ctypes.c_double
        L.or_pairwise_sum.argtypes = [P, ctypes.c_int64]
        L.or_minhash_density.restype = ctypes.c_int64
        L.or_minhash_density.argtypes = [ctypes.c_int64]
        L.or_weight_class.restype = ctypes.c_int
        L.or_weight_class.argtypes = [ctypes.c_double]
        L.or_minhash_csr.restype = ctypes.c_int
        L.or_minhash_csr.argtypes = [P, P, P, P, P, ctypes.c_int64, ctypes.c_int64, P, P, P, P,
                                     ctypes.c_int]
        L.or_lsh_csr.restype = ctypes.c_int
        L.or_lsh_csr.argtypes = [P, P, P, P, P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_int, P, P, P, P, P, ctypes.c_int]
        L.or_darts_flat.restype = ctypes.c_int64
        L.or_darts_flat.argtypes = [P, P, ctypes.c_int64, P, P, ctypes.c_int64, ctypes.c_double,
                                    ctypes.POINTER(ctypes.c_void_p)]
        L.or_free.argtypes = [P]
        L.or_bottom_k.restype = ctypes.c_int
        L.or_bottom_k.argtypes = [P, P, P, P, ctypes.c_int64, ctypes.c_double, ctypes.c_int64,
                                  P, P]
        L.or_hash64_batch.argtypes = [P] * 8 + [ctypes.c_int64, P]
        del u64p
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def tables_for_seed(seed: int) -> np.ndarray:
    """22x256 uint64 tabulation tables: ref/randomness.py:109-110 (numpy MT19937)."""
    rng = np.random.Generator(np.random.MT19937(np.random.SeedSequence(int(seed))))
    return np.ascontiguousarray(rng.integers(0, 2**64, size=(22, 256), dtype=np.uint64))


class Oracle:
    """CPU oracle bound to one hash-family seed."""

    def __init__(self, seed: int):
        self.seed = int(seed)
        self.tables = tables_for_seed(seed)
        self.cdf = np.empty(64, dtype=np.float64)
        lib().or_poisson1_cdf(_p(self.cdf))

    # -- scalar pieces -------------------------------------------------------
    def hash64(self, element, nu=0, rho=0, w=0, r=0, j=0, stream=0) -> int:
        return int(lib().or_hash64(_p(self.tables), element & (2**64 - 1), nu, rho,
                                   w, r, j, stream))

    def hash64_array(self, element, nu, rho, w, r, j, stream) -> np.ndarray:
        cols = [np.ascontiguousarray(np.broadcast_to(np.asarray(c, dtype=np.uint64),
                                                     np.shape(element)))
                for c in (element, nu, rho, w, r, j, stream)]
        out = np.empty(np.shape(element), dtype=np.uint64)
        lib().or_hash64_batch(_p(self.tables), *[_p(c) for c in cols], out.size, _p(out))
        return out

    def mix64(self, values) -> int:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
        return int(lib().or_mix64(_p(self.tables), _p(v), v.size))

    @staticmethod
    def pairwise_sum(a) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64)
        return float(lib().or_pairwise_sum(_p(a), a.size))

    @staticmethod
    def minhash_density(k: int) -> int:
        return int(lib().or_minhash_density(k))

    # -- dart enumeration ------------------------------------------------------
    def darts_below_rank(self, ids, weights, t: int, rank_limit: float):
        """(status, structured array of darts) for one set."""
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = ctypes.c_void_p()
        n = lib().or_darts_flat(_p(self.tables), _p(self.cdf), int(t), _p(ids), _p(w), ids.size,
                                float(rank_limit), ctypes.byref(out))
        if n < 0:
            return int(-n), np.empty(0, dtype=DART_DTYPE)
        if n == 0:
            lib().or_free(out)
            return 0, np.empty(0, dtype=DART_DTYPE)
        buf = (ctypes.c_char * (n * DART_DTYPE.itemsize)).from_address(out.value)
        arr = np.frombuffer(bytes(buf), dtype=DART_DTYPE).copy()
        lib().or_free(out)
        return 0, arr

    def bottom_k(self, ids, weights, k: int):
        """(status, phi, structured array of the k smallest darts) for one set."""
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = np.zeros(k, dtype=DART_DTYPE)
        phi = ctypes.c_int32(0)
        st = lib().or_bottom_k(_p(self.tables), _p(self.cdf), _p(ids), _p(w), ids.size,
                               Oracle.pairwise_sum(w), int(k), _p(out), ctypes.byref(phi))
        return int(st), int(phi.value), out

    # -- batch sketches --------------------------------------------------------
    def minhash_csr(self, indptr, ids, weights, k: int, nthreads: int | None = None):
        indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        n = indptr.size - 1
        out = np.zeros((n, k), dtype=np.uint64)
        status = np.zeros(n, dtype=np.int32)
        phi = np.zeros(n, dtype=np.int32)
        hits = np.zeros(n, dtype=np.int64)
        lib().or_minhash_csr(_p(self.tables), _p(self.cdf), _p(indptr), _p(ids), _p(w), n, k,
                             _p(out), _p(status), _p(phi), _p(hits),
                             nthreads or default_threads())
        return out, status, phi, hits

    def lsh_csr(self, indptr, ids, weights, L: int, K: int, normalize: bool = False,
                want_fps: bool = False, nthreads: int | None = None):
        indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        n = indptr.size - 1
        keys = np.zeros((n, L), dtype=np.uint64)
        fps = np.zeros((n, L, K), dtype=np.uint64) if want_fps else None
        status = np.zeros(n, dtype=np.int32)
        phi = np.zeros(n, dtype=np.int32)
        hits = np.zeros(n, dtype=np.int64)
        lib().or_lsh_csr(_p(self.tables), _p(self.cdf), _p(indptr), _p(ids), _p(w), n, L, K,
                         int(bool(normalize)), _p(keys), _p(fps), _p(status), _p(phi), _p(hits),
                         nthreads or default_threads())
        return keys, fps, status, phi, hits


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)
