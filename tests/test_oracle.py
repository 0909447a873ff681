"""Pin the CPU oracle (oracle/) to the reference's golden vectors.

Every fixture under tests/golden/ was produced by the unmodified reference
package (tests/golden/make_golden.py).  These tests run on CPU only.
"""

import hashlib
import math

import numpy as np
import pytest

from conftest import canonical_darts, golden
from oracle.oracle import Oracle
from paper_2005_11547_b200 import workloads


def csr_digest(indptr, ids, w) -> str:
    h = hashlib.sha256()
    for a in (indptr.astype("<i8"), ids.astype("<u8"), w.astype("<f8")):
        h.update(a.tobytes())
    return h.hexdigest()


def test_golden_hash_value():
    # tests/test_randomness.py:35-39 of the reference
    assert Oracle(1).hash64(123, 4, 5, 6, 7, 8, 9) == 317886004245365293


def test_hash_vectors_all_streams():
    g = golden("hash_vectors.npz")
    orc = Oracle(int(g["seed"]))
    for s_idx, s in enumerate(g["streams"].tolist()):
        got = orc.hash64_array(g["elem"], g["nu"], g["rho"], g["w"], g["r"], g["j"], s)
        assert np.array_equal(got, g["out"][s_idx]), f"stream {s}"


def test_mix64_vectors():
    g = golden("hash_vectors.npz")
    orc = Oracle(int(g["seed"]))
    got = np.array([orc.mix64(row) for row in g["mixseq"]], dtype=np.uint64)
    assert np.array_equal(got, g["mixed"])


def test_poisson_cdf_matches_reference():
    g = golden("hash_vectors.npz")
    orc = Oracle(0)
    assert np.array_equal(orc.cdf, g["cdf"])
    assert (orc.cdf[18:] == 1.0).all()  # counts never exceed 18


def test_minhash_density_and_weight_class():
    g = golden("misc.npz")
    for k, d in zip(g["ks"].tolist(), g["density"].tolist()):
        assert Oracle.minhash_density(k) == d
    # tests/test_core.py:120-123 known answers
    assert Oracle.minhash_density(1) == 1
    assert Oracle.minhash_density(2) == 4
    assert Oracle.minhash_density(256) == 1676
    from oracle.oracle import lib
    for v, c in zip(g["l1s"].tolist(), g["wcs"].tolist()):
        assert lib().or_weight_class(v) == c


def test_pairwise_sum_matches_numpy():
    rng = np.random.default_rng(11)
    sizes = list(range(1, 300)) + [511, 512, 513, 1023, 1024, 1025, 4097, 16384, 20011]
    for n in sizes:
        a = rng.lognormal(0.0, 3.0, n)
        assert Oracle.pairwise_sum(a) == float(np.sum(a)), n


def _check_sweep(name):
    g = golden(name)
    orc = Oracle(int(g["seed"]))
    indptr, ids, w = g["indptr"], g["ids"], g["w"]
    nfull = int(g["full_sets"])
    full = g["full"]
    foff = 0
    for s in range(indptr.size - 1):
        x_ids, x_w = ids[indptr[s]:indptr[s + 1]], w[indptr[s]:indptr[s + 1]]
        l1 = Oracle.pairwise_sum(x_w)
        assert l1 == g["l1"][s]
        limit = float(g["phi"][s]) / l1  # DartHasher.darts, ref/darthash.py:120
        st, darts = orc.darts_below_rank(x_ids, x_w, int(g["t"][s]), limit)
        assert st == 0
        arr = canonical_darts(darts)
        assert arr.size == g["counts"][s], f"set {s}"
        assert hashlib.sha256(arr.tobytes()).hexdigest() == g["digests"][s], f"set {s}"
        if s < nfull:
            assert np.array_equal(arr, full[foff:foff + arr.size])
            foff += arr.size


def test_darts_sweep_criterion1():
    # tests/test_acceptance.py:42-63 sweep, darts tuple-for-tuple
    _check_sweep("darts_sweep.npz")


@pytest.mark.parametrize("tag", ["p64", "m64"])
def test_darts_sweep_extreme_norms(tag):
    # tests/test_acceptance.py:279-284 (||x||_1 = 2^+-64)
    _check_sweep(f"darts_sweep_{tag}.npz")


@pytest.mark.parametrize("name,cfg", [
    ("minhash_cfg1.npz", "cfg1"), ("minhash_cfg2.npz", "cfg2"),
    ("minhash_cfg3_k64.npz", "cfg3"), ("minhash_cfg3_k256.npz", "cfg3"),
    ("minhash_cfg3_k1024.npz", "cfg3"), ("minhash_cfg5.npz", "cfg5")])
def test_minhash_configs(name, cfg):
    g = golden(name)
    rows, k = int(g["rows"]), int(g["k"])
    indptr, ids, w = workloads.generate(cfg, n=rows)
    assert csr_digest(indptr, ids, w) == str(g["digest"]), "workload generator drifted"
    orc = Oracle(workloads.CONFIGS[cfg].seed)
    vals, status, phi, hits = orc.minhash_csr(indptr, ids, w, k)
    assert (status == 0).all()
    assert np.array_equal(vals, g["values"])
    assert np.array_equal(phi, g["phi"])
    assert np.array_equal(hits, g["hits"])
    if "bits" in g.files:
        bits = np.zeros((rows, (k + 63) // 64), dtype=np.uint64)
        for i in range(rows):
            packed = np.packbits((vals[i] & np.uint64(1)).astype(np.uint8), bitorder="little")
            pad = np.zeros(bits.shape[1] * 8, dtype=np.uint8)
            pad[:packed.size] = packed
            bits[i] = pad.view("<u8")
        assert np.array_equal(bits, g["bits"])


def test_minhash_small_and_errors():
    g = golden("minhash_small.npz")
    orc = Oracle(int(g["seed"]))
    for k in g["ks"].tolist():
        vals, status, phi, _ = orc.minhash_csr(g["indptr"], g["ids"], g["w"], k)
        assert np.array_equal(status, g[f"status_k{k}"]), k
        ok = status == 0
        assert np.array_equal(vals[ok], g[f"values_k{k}"][ok]), k
        assert np.array_equal(phi[ok], g[f"phi_k{k}"][ok]), k


def test_lsh_cfg4():
    g = golden("lsh_cfg4.npz")
    rows = int(g["rows"])
    indptr, ids, w = workloads.generate("cfg4", n=rows)
    assert csr_digest(indptr, ids, w) == str(g["digest"])
    orc = Oracle(workloads.CONFIGS["cfg4"].seed)
    keys, fps, status, _, _ = orc.lsh_csr(indptr, ids, w, 100, 20, want_fps=True)
    assert (status == 0).all()
    assert np.array_equal(keys, g["keys"])
    assert np.array_equal(fps[:4], g["fps"])
    nkeys, _, nstatus, _, _ = orc.lsh_csr(indptr, ids, w, 100, 20, normalize=True)
    assert (nstatus == 0).all()
    assert np.array_equal(nkeys, g["norm_keys"])


def test_lsh_small_shapes():
    g = golden("lsh_small.npz")
    orc = Oracle(int(g["seed"]))
    for L, K in ((1, 1), (6, 3), (16, 4), (7, 5)):
        keys, fps, status, _, _ = orc.lsh_csr(g["indptr"], g["ids"], g["w"], L, K, want_fps=True)
        assert (status == 0).all()
        assert np.array_equal(keys, g[f"keys_{L}_{K}"])
        assert np.array_equal(fps, g[f"fps_{L}_{K}"])


def test_lsh_11_equals_minhash_1():
    # tests/test_annindex.py:75-78
    g = golden("lsh_small.npz")
    orc = Oracle(int(g["seed"]))
    _, fps, _, _, _ = orc.lsh_csr(g["indptr"], g["ids"], g["w"], 1, 1, want_fps=True)
    vals, _, _, _ = orc.minhash_csr(g["indptr"], g["ids"], g["w"], 1)
    assert np.array_equal(fps[:, 0, 0], vals[:, 0])
    assert math.isfinite(float(vals.size))


def test_bottom_k_matches_reference():
    # ref/sketching.py:146-156 outputs, tuple for tuple
    g = golden("bottomk_dsk1.npz")
    orc = Oracle(int(g["seed"]))
    indptr = g["indptr"]
    for k in (1, 3, 17, 64):
        exp = g[f"bottomk_k{k}"]
        for s in range(indptr.size - 1):
            st, _, darts = orc.bottom_k(g["ids"][indptr[s]:indptr[s + 1]],
                                        g["w"][indptr[s]:indptr[s + 1]], k)
            assert st == 0
            row = exp[s * k:(s + 1) * k]
            for name in row.dtype.names:
                assert np.array_equal(darts[name], row[name]), (k, s, name)


def test_icws_restatement_matches_reference():
    """A numpy restatement of ICWS (ref/baselines.py:106-136) over the oracle's
    hash reproduces the reference's golden samples (pins the comparator)."""
    g = golden("icws.npz")
    orc = Oracle(int(g["seed"]))
    indptr, ids, w = g["indptr"], g["ids"], g["w"]
    k = 64
    for s in list(range(0, 120, 7)) + list(range(120, indptr.size - 1)):
        x_ids, x_w = ids[indptr[s]:indptr[s + 1]], w[indptr[s]:indptr[s + 1]]
        n = x_ids.size
        elem = np.broadcast_to(x_ids, (k, n))
        coord = np.broadcast_to(np.arange(k, dtype=np.uint64)[:, None], (k, n))

        def u(stream):
            h = orc.hash64_array(elem, 0, 0, coord, 0, 0, stream)
            return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

        r = -(np.log1p(-u(6)) + np.log1p(-u(7)))
        c = -(np.log1p(-u(8)) + np.log1p(-u(9)))
        beta = u(10)
        tick = np.floor(np.log(np.broadcast_to(x_w, (k, n))) / r + beta)
        ln_a = np.log(c) - r * (tick - beta) - r
        win = np.argmin(ln_a, axis=1)
        assert np.array_equal(x_ids[win], g["element_k64"][s]), s
        assert np.array_equal(tick[np.arange(k), win].astype(np.int64), g["tick_k64"][s]), s
