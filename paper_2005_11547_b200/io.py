"""One-line text form of weighted sets (ref/core.py:176-212): space-separated
id:weight tokens, one set per line.  Host-side I/O feeding LshIndex.bulk_load."""

from __future__ import annotations

from .api import WeightedSet, make_weighted_set
from .constants import ValidationError


def format_set(x: WeightedSet) -> str:
    return " ".join(f"{i}:{w!r}" for i, w in zip(x.ids.tolist(), x.weights.tolist()))


def parse_set(line: str) -> WeightedSet:
    pairs = []
    for token in line.split():
        element, sep, weight = token.partition(":")
        if not sep:
            raise ValidationError(f"malformed token {token!r}: expected id:weight")
        try:
            pairs.append((int(element), float(weight)))
        except ValueError:
            raise ValidationError(f"malformed token {token!r}: expected id:weight") from None
    return make_weighted_set(pairs)


def read_sets(path) -> list[WeightedSet]:
    sets = []
    with open(path, "r", encoding="ascii") as handle:
        for lineno, line in enumerate(handle, start=1):
            if not line.strip():
                continue
            try:
                sets.append(parse_set(line))
            except ValidationError as exc:
                raise ValidationError(f"{path}:{lineno}: {exc}") from None
    return sets


def write_sets(path, sets) -> None:
    with open(path, "w", encoding="ascii") as handle:
        for x in sets:
            handle.write(format_set(x) + "\n")
