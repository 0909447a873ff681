"""Host-side constants of a hash family, uploaded once per device.

These are the inputs the reference builds on the host too; the GPU never
recomputes them:
  * tabulation tables: Generator(MT19937(SeedSequence(seed))).integers(
    0, 2**64, (22, 256), uint64)                     ref/randomness.py:109-110
  * Poisson(1) CDF, cdf[0] = exp(-1), term /= n, cdf[63] = 1.0
                                                     ref/randomness.py:66-85
  * floor(log2) thresholds: the reference takes floor(math.log2(y)) for the
    region depths (ref/darthash.py:155-157).  glibc's log2 rounds up to n for
    doubles a few hundred ulps below 2^n, so the device computes the depth as
    e + (y >= thr[e + 1]) with thr[n] = the smallest double below 2^n whose
    host log2 floors to n, probed here from the same libm the reference uses.
  * minhash_density(k) = ceil(k ln k) + k            ref/core.py:150-156
"""

from __future__ import annotations

import math

import numpy as np

KEY_BYTES = 22
POISSON_TABLE_LEN = 64
LOG2_THR_LEN = 258
_PROBE_ULPS = 4096


class ValidationError(ValueError):
    """Raised when input data violates a construction contract (ref/core.py:19-20)."""


def derive_seed(base: int, *indices: int) -> int:
    """A 64-bit seed derived from a base seed and indices (ref/randomness.py:89-92):
    the first word of SeedSequence(base, spawn_key=indices)."""
    seq = np.random.SeedSequence(base, spawn_key=tuple(indices))
    return int(seq.generate_state(1, np.uint64)[0])


def hash_tables(seed: int) -> np.ndarray:
    seed = int(seed)
    if not 0 <= seed <= 2**64 - 1:
        raise ValidationError("seed must fit in 64 bits")  # ref/randomness.py:106-107
    rng = np.random.Generator(np.random.MT19937(np.random.SeedSequence(seed)))
    return np.ascontiguousarray(rng.integers(0, 2**64, size=(KEY_BYTES, 256), dtype=np.uint64))


def poisson1_cdf() -> np.ndarray:
    cdf = np.empty(POISSON_TABLE_LEN, dtype=np.float64)
    term = math.exp(-1.0)
    total = term
    cdf[0] = total
    for n in range(1, POISSON_TABLE_LEN):
        term /= n
        total += term
        cdf[n] = total
    cdf[-1] = 1.0
    return cdf


_LOG2_THR = None


def log2_thresholds() -> np.ndarray:
    """thr[n] for n in [0, 258): smallest y < 2^n with floor(log2(y)) >= n, else 2^n."""
    global _LOG2_THR
    if _LOG2_THR is None:
        thr = np.empty(LOG2_THR_LEN, dtype=np.float64)
        for n in range(LOG2_THR_LEN):
            p = math.ldexp(1.0, n)
            y = p
            steps = 0
            while True:
                below = math.nextafter(y, 0.0)
                if below < 1.0 or math.floor(math.log2(below)) < n:
                    break
                y = below
                steps += 1
                if steps > _PROBE_ULPS:
                    raise RuntimeError(f"log2 round-up region below 2^{n} exceeds probe range")
            thr[n] = y
        _LOG2_THR = thr
    return _LOG2_THR


def floor_log2_via_thresholds(y: float) -> int:
    """Host restatement of the device depth formula (for tests)."""
    thr = log2_thresholds()
    m, e = math.frexp(y)  # y = m * 2^e, m in [0.5, 1)
    e -= 1
    if e >= 256:
        return 1024
    return e + (1 if y >= thr[e + 1] else 0)


def minhash_density(k: int) -> int:
    if k < 1:
        raise ValidationError(f"k must be positive, got {k}")
    if k == 1:
        return 1
    return math.ceil(k * math.log(k)) + k
