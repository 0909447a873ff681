"""Randomised differential soak of the launch variants (GPU vs GPU vs oracle).

Batches large enough for the multi-wave paths (direct-first minhash, the
28-warp direct-only LSH launch) with random k / (L, K), row sizes and weight
scales; every variant must give identical outputs, and a sample of rows is
checked against the C oracle.  usage: python profiles/soak.py [rounds] [seed]
"""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from oracle.oracle import Oracle  # noqa: E402
from paper_2005_11547_b200 import HashFamily, LshParams, as_u64, lsh_batch, minhash_batch  # noqa: E402
from paper_2005_11547_b200 import workloads  # noqa: E402


def batch(rng, n):
    kind = rng.integers(0, 4)
    if kind == 0:
        lens = rng.integers(1, 96, n)
    elif kind == 1:
        lens = np.clip(rng.zipf(1.5, n), 1, 3000)
    elif kind == 2:
        lens = np.full(n, int(rng.integers(8, 200)))
    else:
        lens = rng.integers(1, 12, n)
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=indptr[1:])
    nnz = int(indptr[-1])
    ids = rng.integers(0, 1 << 40, nnz, dtype=np.uint64) * np.uint64(4096) + \
        (np.arange(nnz, dtype=np.uint64) % np.uint64(4096))  # distinct within a row
    scale = 2.0 ** rng.integers(-12, 13)
    w = rng.lognormal(0.0, float(rng.uniform(0.2, 2.0)), nnz) * scale
    if rng.integers(0, 3) == 0:  # a share of normalised rows: rank depth >= 1
        for r in rng.choice(n, n // 3, replace=False):
            w[indptr[r]:indptr[r + 1]] /= w[indptr[r]:indptr[r + 1]].sum()
    return indptr, ids, w


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    bad = 0
    for it in range(rounds):
        n = int(rng.integers(17000, 40000))
        indptr, ids, w = batch(rng, n)
        seed = int(rng.integers(0, 1 << 30))
        fam = HashFamily(seed)
        rows = rng.choice(n, 60, replace=False)
        sp, si, sw = workloads.subset(indptr, ids, w, rows)
        if it % 2 == 0:
            k = int(rng.choice([1, 7, 64, 100, 128, 256, 300]))
            outs = []
            for env in ("0", "1"):
                os.environ["DSK_MH_DIRECT"] = env
                r = minhash_batch(indptr, ids, w, k, fam, bits=True, check=False)
                outs.append((as_u64(r.values), as_u64(r.bits), r.phi.cpu().numpy(),
                             r.status.cpu().numpy()))
            os.environ.pop("DSK_MH_DIRECT")
            same = all(np.array_equal(a, b) for a, b in zip(*outs))
            vals, st, phi, _ = Oracle(seed).minhash_csr(sp, si, sw, k)
            ok = same and np.array_equal(outs[0][0][rows], vals) and \
                np.array_equal(outs[0][2][rows], phi) and np.array_equal(outs[0][3][rows] & 0xFF, st)
            print(f"round {it}: minhash n={n} k={k} nnz={int(indptr[-1])} same={same} oracle_ok={ok} "
                  f"status!=0: {int((outs[0][3] != 0).sum())}", flush=True)
        else:
            L, K = [(100, 20), (16, 8), (9, 3), (40, 33), (128, 4)][int(rng.integers(0, 5))]
            outs = []
            for env in ("1", "0"):
                os.environ["DSK_LSH_DIRECT"] = env
                r = lsh_batch(indptr, ids, w, LshParams(L, K), fam, check=False)
                outs.append((as_u64(r.keys), r.phi.cpu().numpy(), r.status.cpu().numpy()))
            os.environ.pop("DSK_LSH_DIRECT")
            same = all(np.array_equal(a, b) for a, b in zip(*outs))
            keys, _, st, phi, _ = Oracle(seed).lsh_csr(sp, si, sw, L, K)
            ok = same and np.array_equal(outs[0][0][rows], keys) and \
                np.array_equal(outs[0][1][rows], phi) and np.array_equal(outs[0][2][rows] & 0xFF, st)
            print(f"round {it}: lsh n={n} (L,K)=({L},{K}) nnz={int(indptr[-1])} same={same} "
                  f"oracle_ok={ok} status!=0: {int((outs[0][2] != 0).sum())}", flush=True)
        bad += not ok
        torch.cuda.synchronize()
    print("SOAK", "FAILED" if bad else "OK", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
