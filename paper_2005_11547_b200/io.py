"""Text set files <-> CSR batches (the format of ref/core.py:176-212).

A set file holds one weighted set per line as whitespace-separated
`id:weight` tokens; blank lines are skipped.  The reference reads it line by
line into `WeightedSet`s.  Here the whole file becomes one CSR batch
(indptr int64[n+1], ids uint64[nnz], weights float64[nnz]) -- the layout the
GPU entry points take -- so a file of a million sets is sketched in one
launch (`cli sketch`, `LshIndex.bulk_load`).

Validation follows `make_weighted_set` (ref/core.py:69-100): zero weights are
dropped; a malformed token, an id outside [0, 2^64), a non-finite or negative
weight, or a repeated id raises ValidationError naming `path:line` and the
same message the reference gives.  The bulk of the file is checked with
vectorised numpy; only the first offending line is re-checked pair by pair,
to report the reference's message for the first error in file order.
"""

from __future__ import annotations

import math

import numpy as np

from .constants import ValidationError

_U64_MAX = 2**64 - 1


def _token_pair(token: str):
    """(int id, float weight) of one `id:weight` token, or raise."""
    head, colon, tail = token.partition(":")
    if colon:
        try:
            return int(head), float(tail)
        except ValueError:
            pass
    raise ValidationError(f"malformed token {token!r}: expected id:weight")


def _first_pair_error(pairs) -> str | None:
    """The message make_weighted_set raises for these pairs, if any."""
    kept = []
    for element, weight in pairs:
        if element < 0 or element > _U64_MAX:
            return f"element id {element} outside 64-bit range"
        if math.isnan(weight) or math.isinf(weight):
            return f"weight for id {element} is not finite"
        if weight < 0:
            return f"negative weight {weight} for id {element}"
        if weight != 0.0:
            kept.append(element)
    if len(set(kept)) != len(kept):
        return "duplicate element id"
    return None


def parse_line(line: str):
    """(ids uint64[m], weights float64[m]) of one line, zero weights dropped."""
    pairs = [_token_pair(tok) for tok in line.split()]
    err = _first_pair_error(pairs)
    if err:
        raise ValidationError(err)
    keep = [(e, w) for e, w in pairs if w != 0.0]
    return (np.array([e for e, _ in keep], dtype=np.uint64),
            np.array([w for _, w in keep], dtype=np.float64))


def parse_set(line: str):
    """One line as a WeightedSet (ref/core.py:184-195)."""
    from .api import WeightedSet
    ids, weights = parse_line(line)
    return WeightedSet(ids, weights, float(np.sum(weights)) if weights.size else 0.0)


def read_csr(path):
    """Every set of a text file as one CSR batch (indptr, ids, weights)."""
    with open(path, "r", encoding="ascii") as handle:
        lines = handle.read().split("\n")  # universal newlines, as iterating the file
    numbered = [(no, ln) for no, ln in enumerate(lines, start=1) if ln.strip()]
    row_of, elems, wts, malformed = [], [], [], []
    for r, (no, ln) in enumerate(numbered):
        try:
            for tok in ln.split():
                e, w = _token_pair(tok)
                elems.append(e)
                wts.append(w)
                row_of.append(r)
        except ValidationError:
            malformed.append(r)
    n = len(numbered)
    rows = np.asarray(row_of, dtype=np.int64)
    w = np.asarray(wts, dtype=np.float64)
    in_range = np.fromiter((0 <= e <= _U64_MAX for e in elems), dtype=bool, count=len(elems))
    bad_pair = ~in_range | ~np.isfinite(w) | (w < 0)
    keep = (w != 0.0) & ~bad_pair
    ids = np.zeros(len(elems), dtype=np.uint64)
    if in_range.any():
        ids[in_range] = np.array([e for e, ok in zip(elems, in_range) if ok], dtype=np.uint64)
    # rows repeating a kept id: sort (row, id) pairs
    kr, ki = rows[keep], ids[keep]
    order = np.lexsort((ki, kr))
    sr, si = kr[order], ki[order]
    dup_rows = sr[1:][(sr[1:] == sr[:-1]) & (si[1:] == si[:-1])]
    bad_rows = np.union1d(np.union1d(np.unique(rows[bad_pair]), dup_rows),
                          np.asarray(malformed, dtype=np.int64))
    if bad_rows.size:  # the reference stops at the first bad line, in file order
        no, ln = numbered[int(bad_rows[0])]
        try:
            parse_line(ln)
        except ValidationError as exc:
            raise ValidationError(f"{path}:{no}: {exc}") from None
    lengths = np.bincount(kr, minlength=n).astype(np.int64)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lengths, out=indptr[1:])
    return indptr, np.ascontiguousarray(ids[keep]), np.ascontiguousarray(w[keep])


def read_sets(path) -> list:
    """Every set of a text file as WeightedSets (ref/core.py:198-206)."""
    from .api import WeightedSet
    indptr, ids, w = read_csr(path)
    out = []
    for r in range(indptr.size - 1):
        a, b = int(indptr[r]), int(indptr[r + 1])
        out.append(WeightedSet(ids[a:b], w[a:b], float(np.sum(w[a:b])) if b > a else 0.0))
    return out


def format_line(ids, weights) -> str:
    """The text form of one set: `id:repr(weight)` tokens (ref/core.py:178-181)."""
    return " ".join(f"{int(e)}:{float(x)!r}" for e, x in zip(ids, weights))


def format_set(x) -> str:
    return format_line(x.ids.tolist(), x.weights.tolist())


def write_csr(path, indptr, ids, weights) -> None:
    """Write a CSR batch as a set file, one line per row."""
    ids_l, w_l = np.asarray(ids).tolist(), np.asarray(weights).tolist()
    bounds = np.asarray(indptr).tolist()
    with open(path, "w", encoding="ascii") as handle:
        for r in range(len(bounds) - 1):
            handle.write(format_line(ids_l[bounds[r]:bounds[r + 1]],
                                     w_l[bounds[r]:bounds[r + 1]]) + "\n")


def write_sets(path, sets) -> None:
    with open(path, "w", encoding="ascii") as handle:
        for x in sets:
            handle.write(format_set(x) + "\n")
