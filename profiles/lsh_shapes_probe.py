"""Multi-wave LSH batches at unusual (L, K): GPU (default shape choice) vs the general path vs the oracle."""
import os, sys
import numpy as np, torch
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from oracle.oracle import Oracle
from paper_2005_11547_b200 import HashFamily, LshParams, as_u64, lsh_batch, workloads
bad = 0
for (L, K, n, wl) in [(2000, 2, 20000, "cfg3"), (8, 1, 40000, "cfg3"), (7, 3, 40000, "cfg3"), (300, 5, 20000, "cfg4"),
                      (1, 30, 30000, "cfg3"), (1200, 1, 20000, "cfg5"), (100, 20, 17000, "cfg5"), (64, 32, 20000, "cfg4")]:
    indptr, ids, w = workloads.generate(wl, n=n, start=123)
    f = HashFamily(9)
    outs = []
    for env in ("1", "0"):
        os.environ["DSK_LSH_DIRECT"] = env
        r = lsh_batch(indptr, ids, w, LshParams(L, K), f, check=False)
        outs.append((as_u64(r.keys), r.phi.cpu().numpy(), r.status.cpu().numpy()))
    os.environ.pop("DSK_LSH_DIRECT")
    same = all(np.array_equal(a, b) for a, b in zip(*outs))
    rows = np.arange(0, n, n // 25)
    sp, si, sw = workloads.subset(indptr, ids, w, rows)
    keys, _, st, phi, _ = Oracle(9).lsh_csr(sp, si, sw, L, K)
    ok = same and np.array_equal(outs[0][0][rows], keys) and np.array_equal(outs[0][1][rows], phi) and np.array_equal(outs[0][2][rows] & 0xFF, st)
    print(f"(L,K)=({L},{K}) n={n} {wl}: same={same} oracle_ok={ok} status!=0: {int((outs[0][2] != 0).sum())}", flush=True)
    bad += not ok
print("PROBE", "FAILED" if bad else "OK")
sys.exit(1 if bad else 0)
