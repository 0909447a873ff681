"""The reference's running-time shape criteria, re-run on the GPU batch path.

    python profiles/acceptance_shapes.py [--sets 4096] > profiles/r02/acceptance_shapes.json

/root/reference/pkg/tests/test_acceptance.py:229-277 (criteria 7 and 8; SPEC.md
:538-539) times single sets on one CPU core.  Here every cell is one batch of
`--sets` sets of the cell's shape, generated as ref/bench.py:82-100 does
(distinct uniform 64-bit ids, weights a uniform draw from the simplex scaled
to l1), sketched by one launch of the batch kernel with the inputs resident
in HBM; per-set time = median batch time / sets.  Criteria:

  7a  ICWS / DartMinHash time >= 2 at (k, l0) = (256, 256) and (1024, 1024)
  7b  DartMinHash time growth l0 = 64 -> 16384 at k = 1024 <= 16
  7c  ICWS ms / (k * l0) spread over k in {64, 256} x l0 in {256, 1024, 4096} <= 2
  8   DartMinHash slowdown at ||x||_1 = 2^64 and 2^-64 vs 1 (k = 256, l0 = 1024) >= 5
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2005_11547_b200 import HashFamily, icws_batch, minhash_batch  # noqa: E402


def gen_batch(n, l0, l1, seed):
    """n sets shaped like ref/bench.py:gen_set (distinct ids, simplex weights * l1)."""
    rng = np.random.Generator(np.random.MT19937(np.random.SeedSequence(seed)))
    ids = rng.integers(0, 2**64, size=(n, l0), dtype=np.uint64)
    srt = np.sort(ids, axis=1)
    assert not (srt[:, 1:] == srt[:, :-1]).any()  # 64-bit ids: collisions ~ never
    expo = -np.log1p(-rng.random((n, l0)))
    w = expo / expo.sum(axis=1, keepdims=True) * l1
    indptr = np.arange(n + 1, dtype=np.int64) * l0
    return indptr, ids.reshape(-1), w.reshape(-1)


def cell_ms(algo, k, l0, l1, n, seed, reps=5):
    dev = torch.device("cuda", 0)
    indptr, ids, w = gen_batch(n, l0, l1, seed)
    p = torch.from_numpy(indptr).to(dev)
    i = torch.from_numpy(ids.view(np.int64)).to(dev)
    ww = torch.from_numpy(w).to(dev)
    fam = HashFamily(seed)

    def run():
        if algo == "dartminhash":
            return minhash_batch(p, i, ww, k, fam, check=False)
        return icws_batch(p, i, ww, k, fam, check=False)

    for _ in range(2):
        res = run()
    torch.cuda.synchronize()
    assert int((res.status != 0).sum()) == 0, (algo, k, l0, l1)
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    return statistics.median(times) / n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", type=int, default=4096)
    args = ap.parse_args()
    n = args.sets
    out = {"sets_per_cell": n, "method": "one batch launch per cell, device-resident, median of 5",
           "cells_ms_per_set": {}, "criteria": {}}
    t = out["cells_ms_per_set"]

    def cell(algo, k, l0, l1, seed):
        key = f"{algo} k={k} l0={l0} l1={l1:g}"
        t[key] = cell_ms(algo, k, l0, l1, n, seed)
        return t[key]

    r1 = cell("icws", 256, 256, 1.0, 0xC7A) / cell("dartminhash", 256, 256, 1.0, 0xC7A)
    r2 = cell("icws", 1024, 1024, 1.0, 0xC7A) / cell("dartminhash", 1024, 1024, 1.0, 0xC7A)
    out["criteria"]["7a_icws_over_dart"] = {"k256_l0_256": r1, "k1024_l0_1024": r2,
                                             "need": ">= 2", "pass": r1 >= 2 and r2 >= 2}
    g = cell("dartminhash", 1024, 16384, 1.0, 0xC7B) / cell("dartminhash", 1024, 64, 1.0, 0xC7B)
    out["criteria"]["7b_dart_l0_growth_64_to_16384"] = {"growth": g, "need": "<= 16",
                                                         "pass": g <= 16}
    per = []
    for k in (64, 256):
        for l0 in (256, 1024, 4096):
            per.append(cell("icws", k, l0, 1.0, 0xC7C) / (k * l0))
    spread = max(per) / min(per)
    out["criteria"]["7c_icws_linear_spread"] = {"spread": spread, "need": "<= 2",
                                                "pass": spread <= 2}
    base = cell("dartminhash", 256, 1024, 1.0, 0xC8)
    up = cell("dartminhash", 256, 1024, 2.0**64, 0xC8) / base
    down = cell("dartminhash", 256, 1024, 2.0**-64, 0xC8) / base
    out["criteria"]["8_extreme_norm_slowdown"] = {"2^64": up, "2^-64": down, "need": ">= 5",
                                                  "pass": up >= 5 and down >= 5}
    out["all_pass"] = all(c["pass"] for c in out["criteria"].values())
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
