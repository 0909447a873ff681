"""Parity report over the subsets SURVEY.md §8(d) prescribes (GPU box).

    python tests/parity_report.py [--out profiles/r02/parity_report.json]

For every configuration the GPU sketches the FULL population (device
resident, one launch per config / k), then the C oracle (oracle/, the
pinned restatement of the reference) recomputes a deterministic subset on
all host cores and the two are compared slot for slot:

  cfg1  all 1,000 rows (k = 64, + 1-bit words)
  cfg2  all 100,000 rows (k = 256)
  cfg3  every 100th row of 1e6, for k = 64, 256 and 1024, values + 1-bit words
  cfg4  every 100th row of 1e6, the 100 LSH keys (lsh_key + mix64 per table)
  cfg5  every 100th row of 1e7, plus every row with nnz >= 4096 (k = 128)

Reported per config: rows checked, slots checked, mismatching slots (split
into rows flagged DSK_STATUS_TIE -- bit-identical fp64 ranks, the only
mismatch the north star tolerates, budget 1e-6 of slots -- and unflagged),
phi* disagreements, status != 0 rows, and the hit count H(phi*) agreement.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle.oracle import Oracle, default_threads  # noqa: E402  (test infrastructure)
from paper_2005_11547_b200 import (DSK_STATUS_TIE, HashFamily, LshParams, as_u64,  # noqa: E402
                                   lsh_batch, minhash_batch, workloads)


def pack_bits(vals: np.ndarray, k: int) -> np.ndarray:
    words = (k + 63) // 64
    out = np.zeros((vals.shape[0], words), dtype=np.uint64)
    for j in range(k):
        out[:, j // 64] |= (vals[:, j] & np.uint64(1)) << np.uint64(j % 64)
    return out


def compare(name, got, want, status, phi_g, phi_o, st_o, hits_g=None, hits_o=None):
    tie_rows = (status & DSK_STATUS_TIE) != 0
    diff = got != want
    slots = int(diff.size)
    mism = int(diff.sum())
    mism_tie = int(diff[tie_rows].sum()) if tie_rows.any() else 0
    rep = {"rows": int(got.shape[0]), "slots": slots, "mismatching_slots": mism,
           "mismatching_slots_in_tie_rows": mism_tie,
           "mismatching_slots_unflagged": mism - mism_tie,
           "tie_rows": int(tie_rows.sum()), "tie_budget_slots": slots * 1e-6,
           "phi_mismatch_rows": int((phi_g != phi_o).sum()),
           "status_nonzero_gpu": int(((status & 0xFF) != 0).sum()),
           "status_nonzero_oracle": int((st_o != 0).sum())}
    if hits_g is not None:
        rep["hits_mismatch_rows"] = int((hits_g != hits_o).sum())
    rep["bit_exact"] = mism == 0 and rep["phi_mismatch_rows"] == 0 and \
        rep["status_nonzero_gpu"] == rep["status_nonzero_oracle"] == 0
    print(f"{name}: {json.dumps(rep)}", flush=True)
    return rep


def minhash_case(name, cfg, k, rows_sel, orc, threads, full=None, bits=False):
    t0 = time.time()
    indptr, ids, w = full if full is not None else workloads.generate(cfg)
    res = minhash_batch(indptr, ids, w, k, HashFamily(workloads.CONFIGS[cfg].seed), bits=bits,
                        check=False, device="cuda:0")
    sel = rows_sel(indptr)
    sel_d = torch.from_numpy(sel).to(res.values.device)
    vals = as_u64(res.values[sel_d])  # gather on the device (cfg5: 10 GB of values)
    status = res.status.cpu().numpy()[sel]
    phi_g = res.phi.cpu().numpy()[sel]
    hits_g = res.stats.cpu().numpy().view(np.uint32)[sel, 2].astype(np.int64)
    t_gpu = time.time() - t0
    sp, si, sw = workloads.subset(indptr, ids, w, sel)
    t1 = time.time()
    ov, ost, ophi, ohits = orc.minhash_csr(sp, si, sw, k, nthreads=threads)
    rep = compare(name, vals, ov, status, phi_g, ophi, ost, hits_g, ohits)
    if bits:
        gb = as_u64(res.bits[sel_d])
        rep["onebit_word_mismatches"] = int((gb != pack_bits(ov, k)).sum())
        rep["bit_exact"] = rep["bit_exact"] and rep["onebit_word_mismatches"] == 0
    rep.update({"population": int(indptr.size - 1), "k": k, "gpu_s": round(t_gpu, 2),
                "oracle_s": round(time.time() - t1, 2)})
    return rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(REPO, "profiles", "r02", "parity_report.json"))
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))
    threads = default_threads()
    report = {"oracle_threads": threads, "configs": {}}
    every = lambda step: (lambda p: np.arange(0, p.size - 1, step))  # noqa: E731

    def want(tag):
        return not only or tag in only

    if want("cfg1"):
        report["configs"]["cfg1"] = minhash_case("cfg1", "cfg1", 64, every(1), Oracle(0), threads,
                                                 bits=True)
        report["configs"]["cfg1"]["subset"] = "all rows"
    if want("cfg2"):
        report["configs"]["cfg2"] = minhash_case("cfg2", "cfg2", 256, every(1), Oracle(1), threads)
        report["configs"]["cfg2"]["subset"] = "all rows"
    if want("cfg3"):
        full = workloads.generate("cfg3")
        for k in (64, 256, 1024):
            tag = f"cfg3_k{k}"
            report["configs"][tag] = minhash_case(tag, "cfg3", k, every(100), Oracle(2), threads,
                                                  full=full, bits=True)
            report["configs"][tag]["subset"] = "every 100th row"
        del full
    if want("cfg4"):
        t0 = time.time()
        cfg = workloads.CONFIGS["cfg4"]
        indptr, ids, w = workloads.generate("cfg4")
        res = lsh_batch(indptr, ids, w, LshParams(cfg.L, cfg.K), HashFamily(cfg.seed),
                        check=False, device="cuda:0")
        sel = np.arange(0, indptr.size - 1, 100)
        keys = as_u64(res.keys)[sel]
        status = res.status.cpu().numpy()[sel]
        phi_g = res.phi.cpu().numpy()[sel]
        hits_g = res.stats.cpu().numpy().view(np.uint32)[sel, 2].astype(np.int64)
        t_gpu = time.time() - t0
        sp, si, sw = workloads.subset(indptr, ids, w, sel)
        t1 = time.time()
        okeys, _, ost, ophi, ohits = Oracle(cfg.seed).lsh_csr(sp, si, sw, cfg.L, cfg.K,
                                                               nthreads=threads)
        rep = compare("cfg4", keys, okeys, status, phi_g, ophi, ost, hits_g, ohits)
        rep.update({"population": int(indptr.size - 1), "L": cfg.L, "K": cfg.K,
                    "subset": "every 100th row", "gpu_s": round(t_gpu, 2),
                    "oracle_s": round(time.time() - t1, 2)})
        report["configs"]["cfg4"] = rep
        del indptr, ids, w, res
    if want("cfg5"):
        def cfg5_rows(p):
            nnz = np.diff(p)
            return np.union1d(np.arange(0, p.size - 1, 100), np.nonzero(nnz >= 4096)[0])
        rep = minhash_case("cfg5", "cfg5", 128, cfg5_rows, Oracle(4), threads)
        rep["subset"] = "every 100th row plus every row with nnz >= 4096"
        report["configs"]["cfg5"] = rep
    report["all_bit_exact"] = all(r["bit_exact"] for r in report["configs"].values())
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(report, open(args.out, "w"), indent=1)
    print(json.dumps({"all_bit_exact": report["all_bit_exact"]}))


if __name__ == "__main__":
    main()
