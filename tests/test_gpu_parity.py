"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the CPU oracle.  Bit-exact for every integer output
(fingerprints, packed bits, keys, dart tuples); fp64 dart weights/ranks are
compared bit-for-bit too (the reference's rounding order is reproduced).
"""

import hashlib

import numpy as np
import pytest
import torch

from conftest import canonical_darts, golden
from oracle.oracle import Oracle
from paper_2005_11547_b200 import (
    DSK_STATUS_TIE,
    DartHasher,
    HashFamily,
    LshParams,
    ValidationError,
    WeightedSet,
    as_u64,
    dart_minhash,
    darts_batch,
    lsh_batch,
    lsh_key,
    make_weighted_set,
    minhash_batch,
    minhash_density,
    one_bit,
    workloads,
)

pytestmark = pytest.mark.gpu

_FAMILIES = {}


def fam(seed):
    if seed not in _FAMILIES:
        _FAMILIES[seed] = HashFamily(seed)
    return _FAMILIES[seed]


def csr_digest(indptr, ids, w) -> str:
    h = hashlib.sha256()
    for a in (indptr.astype("<i8"), ids.astype("<u8"), w.astype("<f8")):
        h.update(a.tobytes())
    return h.hexdigest()


def test_cuda_available():
    assert torch.cuda.is_available()
    major, minor = torch.cuda.get_device_capability()
    assert (major, minor) >= (10, 0)


def test_hash64_golden():
    # tests/test_randomness.py:35-39 of the reference
    assert fam(1).hash64(123, 4, 5, 6, 7, 8, 9) == 317886004245365293


def test_hash64_vectors_all_streams():
    g = golden("hash_vectors.npz")
    f = fam(int(g["seed"]))
    for s_idx, s in enumerate(g["streams"].tolist()):
        got = f.hash64_array(g["elem"], g["nu"], g["rho"], g["w"], g["r"], g["j"], s)
        assert np.array_equal(got, g["out"][s_idx]), f"stream {s}"


def test_mix64_vectors():
    g = golden("hash_vectors.npz")
    f = fam(int(g["seed"]))
    assert np.array_equal(f.mix64_rows(g["mixseq"]), g["mixed"])
    assert f.mix64(g["mixseq"][0].tolist()) == int(g["mixed"][0])


def _gpu_darts_sweep(name):
    g = golden(name)
    f = fam(int(g["seed"]))
    indptr, ids, w = g["indptr"], g["ids"], g["w"]
    n = indptr.size - 1
    limits = g["phi"] / g["l1"]  # DartHasher.darts: phi / ||x||_1
    mism = 0
    # the kernel takes one t per call: group rows by t
    for t in np.unique(g["t"]).tolist():
        rows = np.nonzero(g["t"] == t)[0]
        sp, si, sw = workloads.subset(indptr, ids, w, rows)
        offsets, status, cols = darts_batch(sp, si, sw, t, limits[rows], f)
        assert (status.cpu().numpy() == 0).all()
        off = offsets.cpu().numpy()
        host = {k: v.cpu().numpy() for k, v in cols.items()}
        for q, s in enumerate(rows.tolist()):
            a, b = off[q], off[q + 1]
            arr = np.empty(b - a, dtype=[("element", "<u8"), ("nu", "<u2"), ("rho", "<u2"),
                                         ("w", "<u4"), ("r", "<u4"), ("j", "<u2"),
                                         ("weight", "<f8"), ("rank", "<f8"),
                                         ("fingerprint", "<u8")])
            arr["element"] = host["element"][a:b].view(np.uint64)
            arr["nu"] = host["nu"][a:b].view(np.uint16)
            arr["rho"] = host["rho"][a:b].view(np.uint16)
            arr["w"] = host["w"][a:b].view(np.uint32)
            arr["r"] = host["r"][a:b].view(np.uint32)
            arr["j"] = host["j"][a:b].view(np.uint16)
            arr["weight"] = host["weight"][a:b]
            arr["rank"] = host["rank"][a:b]
            arr["fingerprint"] = host["fingerprint"][a:b].view(np.uint64)
            c = canonical_darts(arr)
            if c.size != g["counts"][s] or \
                    hashlib.sha256(c.tobytes()).hexdigest() != g["digests"][s]:
                mism += 1
    assert mism == 0, f"{mism}/{n} sets differ"


def test_darts_criterion1_sweep():
    # tests/test_acceptance.py:42-63: 1000 sets, l0 <= 64, norms 2^+-4,
    # phi in {.5,1,2,4}, t in {1,16,256}: tuple-for-tuple equal
    _gpu_darts_sweep("darts_sweep.npz")


@pytest.mark.parametrize("tag", ["p64", "m64"])
def test_darts_extreme_norms(tag):
    # tests/test_acceptance.py:279-284
    _gpu_darts_sweep(f"darts_sweep_{tag}.npz")


@pytest.mark.parametrize("name,cfg", [
    ("minhash_cfg1.npz", "cfg1"), ("minhash_cfg2.npz", "cfg2"),
    ("minhash_cfg3_k64.npz", "cfg3"), ("minhash_cfg3_k256.npz", "cfg3"),
    ("minhash_cfg3_k1024.npz", "cfg3"), ("minhash_cfg5.npz", "cfg5")])
def test_minhash_golden(name, cfg):
    g = golden(name)
    rows, k = int(g["rows"]), int(g["k"])
    indptr, ids, w = workloads.generate(cfg, n=rows)
    assert csr_digest(indptr, ids, w) == str(g["digest"])
    res = minhash_batch(indptr, ids, w, k, fam(workloads.CONFIGS[cfg].seed),
                        bits="bits" in g.files)
    assert (res.status.cpu().numpy() == 0).all()
    assert np.array_equal(as_u64(res.values), g["values"])
    assert np.array_equal(res.phi.cpu().numpy(), g["phi"])
    st = res.stats.cpu().numpy().view(np.uint32)
    assert np.array_equal(st[:, 2].astype(np.int64), g["hits"])  # H(phi*) per set
    if "bits" in g.files:
        assert np.array_equal(as_u64(res.bits), g["bits"])


def test_minhash_small_edge_cases():
    g = golden("minhash_small.npz")
    f = fam(int(g["seed"]))
    for k in g["ks"].tolist():
        res = minhash_batch(g["indptr"], g["ids"], g["w"], k, f, check=False)
        status = res.status.cpu().numpy()
        assert np.array_equal(status & 0xFF, g[f"status_k{k}"]), k
        assert not (status & DSK_STATUS_TIE).any()
        ok = status == 0
        assert np.array_equal(as_u64(res.values)[ok], g[f"values_k{k}"][ok]), k
        assert np.array_equal(res.phi.cpu().numpy()[ok], g[f"phi_k{k}"][ok]), k


def _oracle_compare(cfg, k, rows, start=0, bits=False):
    indptr, ids, w = workloads.generate(cfg, n=rows, start=start)
    seed = workloads.CONFIGS[cfg].seed
    res = minhash_batch(indptr, ids, w, k, fam(seed), bits=bits)
    vals, status, phi, hits = Oracle(seed).minhash_csr(indptr, ids, w, k)
    assert (status == 0).all()
    gv = as_u64(res.values)
    mism = int((gv != vals).sum())
    assert mism == 0, f"{cfg} k={k}: {mism} slot mismatches of {vals.size}"
    assert np.array_equal(res.phi.cpu().numpy(), phi)
    assert np.array_equal(res.stats.cpu().numpy().view(np.uint32)[:, 2].astype(np.int64), hits)
    if bits:
        ob = np.zeros((rows, (k + 63) // 64), dtype=np.uint64)
        for i in range(rows):
            packed = np.packbits((vals[i] & np.uint64(1)).astype(np.uint8), bitorder="little")
            pad = np.zeros(ob.shape[1] * 8, dtype=np.uint8)
            pad[:packed.size] = packed
            ob[i] = pad.view("<u8")
        assert np.array_equal(as_u64(res.bits), ob)


def test_minhash_cfg2_vs_oracle():
    _oracle_compare("cfg2", 256, 1500, start=3000)


@pytest.mark.parametrize("k", [64, 256, 1024])
def test_minhash_cfg3_vs_oracle(k):
    _oracle_compare("cfg3", k, {64: 4000, 256: 2000, 1024: 600}[k], start=70000, bits=True)


def _ragged_batch(seed, lens, sigma=2.0, d=1 << 26):
    rng = np.random.default_rng(seed)
    lens = np.asarray(lens, dtype=np.int64)
    indptr = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    ids = np.concatenate([rng.choice(d, int(m), replace=False).astype(np.uint64) if m else
                          np.zeros(0, np.uint64) for m in lens])
    w = rng.lognormal(0.0, sigma, int(indptr[-1]))
    return indptr, ids, w


def test_minhash_max_sizes_and_ragged_vs_oracle():
    """cfg5's extremes: sets at its nnz clip (16384) and beyond, single-element
    and empty sets in one ragged batch (per-set status for the empty ones)."""
    lens = [16384, 0, 1, 16384, 2, 3000, 0, 65536, 1, 16383, 7, 16385]
    indptr, ids, w = _ragged_batch(21, lens)
    for k in (1, 128, 300):
        res = minhash_batch(indptr, ids, w, k, fam(4), check=False)
        vals, status, phi, hits = Oracle(4).minhash_csr(indptr, ids, w, k)
        st = res.status.cpu().numpy()
        assert np.array_equal(st, status), k
        ok = status == 0
        assert ok.sum() == len(lens) - 2
        assert np.array_equal(as_u64(res.values)[ok], vals[ok]), k
        assert np.array_equal(res.phi.cpu().numpy()[ok], phi[ok]), k
        got_h = res.stats.cpu().numpy().view(np.uint32)[:, 2].astype(np.int64)
        assert np.array_equal(got_h[ok], hits[ok]), k


@pytest.mark.parametrize("k", [5000, 12000])
def test_minhash_large_k_global_slots_vs_oracle(k):
    """k beyond the shared-memory slot array: slots live in global memory."""
    indptr, ids, w = workloads.generate("cfg1", n=6)
    res = minhash_batch(indptr, ids, w, k, fam(0), bits=True)
    vals, status, phi, hits = Oracle(0).minhash_csr(indptr, ids, w, k)
    assert (status == 0).all()
    assert np.array_equal(as_u64(res.values), vals)
    assert np.array_equal(res.phi.cpu().numpy(), phi)
    assert np.array_equal(res.stats.cpu().numpy().view(np.uint32)[:, 2].astype(np.int64), hits)
    packed = np.packbits((vals & np.uint64(1)).astype(np.uint8), axis=1, bitorder="little")
    pad = np.zeros((6, ((k + 63) // 64) * 8), dtype=np.uint8)
    pad[:, :packed.shape[1]] = packed
    assert np.array_equal(as_u64(res.bits), pad.view("<u8"))


def test_lsh_max_sizes_vs_oracle():
    lens = [16384, 1, 4000, 16384, 2, 20000]
    indptr, ids, w = _ragged_batch(22, lens, sigma=1.0)
    res = lsh_batch(indptr, ids, w, LshParams(100, 20), fam(3), fps=True)
    keys, fps, status, phi, _ = Oracle(3).lsh_csr(indptr, ids, w, 100, 20, want_fps=True)
    assert (status == 0).all()
    assert np.array_equal(as_u64(res.keys), keys)
    assert np.array_equal(as_u64(res.fps), fps)
    assert np.array_equal(res.phi.cpu().numpy(), phi)


@pytest.mark.parametrize("cfg,k,rows", [("cfg2", 256, 100000), ("cfg3", 256, 100000),
                                         ("cfg5", 128, 100000)])
def test_minhash_full_size_vs_oracle(cfg, k, rows):
    """Every slot of BASELINE-sized batches (cfg2 is its full 1e5 sets)
    against the oracle: zero mismatching slots (north star: <= 1e-6)."""
    _oracle_compare(cfg, k, rows)


def test_lsh_large_batch_vs_oracle():
    indptr, ids, w = workloads.generate("cfg4", n=30000, start=40000)
    res = lsh_batch(indptr, ids, w, LshParams(100, 20), fam(3))
    keys, _, status, phi, hits = Oracle(3).lsh_csr(indptr, ids, w, 100, 20)
    assert (status == 0).all()
    assert int((as_u64(res.keys) != keys).sum()) == 0
    assert np.array_equal(res.phi.cpu().numpy(), phi)


def test_minhash_cfg5_vs_oracle():
    _oracle_compare("cfg5", 128, 4000, start=200000)


def test_minhash_cfg5_largest_first_order_vs_oracle():
    # 20000 heavy-tailed rows span several waves of teams: the launch
    # processes them largest size class first (outputs stay in row order)
    _oracle_compare("cfg5", 128, 20000, start=500000)


def test_minhash_odd_k_vs_oracle():
    # non-power-of-two bucket counts exercise the 64-bit modulo
    for k in (1, 3, 100, 333, 2000):
        _oracle_compare("cfg1", k, 60)


def test_minhash_determinism_and_row_order():
    indptr, ids, w = workloads.generate("cfg3", n=3000)
    f = fam(2)
    a = as_u64(minhash_batch(indptr, ids, w, 256, f).values)
    b = as_u64(minhash_batch(indptr, ids, w, 256, f).values)
    assert np.array_equal(a, b)
    rows = np.random.default_rng(5).permutation(3000)
    sp, si, sw = workloads.subset(indptr, ids, w, rows)
    c = as_u64(minhash_batch(sp, si, sw, 256, f).values)
    assert np.array_equal(c, a[rows])
    # element order inside a set does not matter (total order on darts)
    perm_rows = []
    for r in range(50):
        seg = np.arange(indptr[r], indptr[r + 1])
        perm_rows.append(np.random.default_rng(r).permutation(seg))
    take = np.concatenate(perm_rows)
    pp = indptr[:51].copy()
    d = as_u64(minhash_batch(pp, ids[take], w[take], 256, f).values)
    assert np.array_equal(d, a[:50])


def test_facade_single_set_api():
    f = fam(0xBEEF)
    x = make_weighted_set([(1, 0.5), (2, 0.25), (3, 1.25)])
    # k = 1 equals the global (rank, index)-minimum dart (tests/test_sketching.py:42-46)
    darts = DartHasher(1, f).darts(x, 64.0)
    best = min(darts, key=lambda d: (d.rank, d.index))
    assert dart_minhash(x, 1, f).values.tolist() == [best.fingerprint]
    s = dart_minhash(x, 64, f)
    assert one_bit(s).bits.tolist() == (s.values & np.uint64(1)).tolist()
    with pytest.raises(ValidationError):
        dart_minhash(make_weighted_set([]), 4, f)
    with pytest.raises(ValidationError):
        dart_minhash(x, 0, f)
    # darts against the oracle
    orc = Oracle(0xBEEF)
    st, od = orc.darts_below_rank(x.ids, x.weights, 16, 3.0)
    gd = DartHasher(16, f).darts_below_rank(x, 3.0)
    assert st == 0 and len(gd) == od.size
    assert {d.index for d in gd} == {(int(e), int(a), int(b), int(c), int(r), int(j))
                                     for e, a, b, c, r, j in zip(od["element"], od["nu"], od["rho"],
                                                                 od["w"], od["r"], od["j"])}


def test_batch_status_errors():
    f = fam(3)
    indptr = np.array([0, 1, 1, 3, 4], dtype=np.int64)
    ids = np.array([5, 6, 7, 8], dtype=np.uint64)
    w = np.array([1.0, 0.5, -1.0, np.inf])
    res = minhash_batch(indptr, ids, w, 16, f, check=False)
    assert res.status.cpu().numpy().tolist() == [0, 1, 2, 2]
    with pytest.raises(ValidationError):
        minhash_batch(indptr, ids, w, 16, f)


def test_minhash_density_matches():
    for k in (1, 2, 64, 128, 256, 1024, 2000):
        assert minhash_density(k) == Oracle.minhash_density(k)


def test_host_buffer_abi_matches_device_path():
    """dsk_minhash_csr_host (numpy buffers, chunked pipeline) == device path."""
    import ctypes

    from paper_2005_11547_b200 import _lib
    indptr, ids, w = workloads.generate("cfg2", n=9000)
    f = fam(1)
    k = 256
    dev = minhash_batch(indptr, ids, w, k, f, bits=True)
    vals = np.zeros((9000, k), dtype=np.uint64)
    bits = np.zeros((9000, 4), dtype=np.uint64)
    status = np.zeros(9000, dtype=np.int32)
    phi = np.zeros(9000, dtype=np.int32)
    stats = np.zeros((9000, 4), dtype=np.uint32)
    P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    rc = _lib.load().dsk_minhash_csr_host(f.context(), P(indptr), P(ids), P(w), 9000, k, P(vals),
                                         P(bits), P(status), P(phi), P(stats))
    assert rc == 0
    assert (status == 0).all()
    assert np.array_equal(vals, as_u64(dev.values))
    assert np.array_equal(bits, as_u64(dev.bits))
    assert np.array_equal(phi, dev.phi.cpu().numpy())
    assert np.array_equal(stats, dev.stats.cpu().numpy().view(np.uint32))


# ------------------------------------------------------------------ LSH (K5)


def test_lsh_cfg4_golden():
    g = golden("lsh_cfg4.npz")
    rows = int(g["rows"])
    indptr, ids, w = workloads.generate("cfg4", n=rows)
    assert csr_digest(indptr, ids, w) == str(g["digest"])
    f = fam(workloads.CONFIGS["cfg4"].seed)
    res = lsh_batch(indptr, ids, w, LshParams(100, 20), f, fps=True)
    assert np.array_equal(as_u64(res.keys), g["keys"])
    assert np.array_equal(as_u64(res.fps)[:4], g["fps"])
    nres = lsh_batch(indptr, ids, w, LshParams(100, 20), f, normalize=True)
    assert np.array_equal(as_u64(nres.keys), g["norm_keys"])


def test_lsh_small_shapes():
    g = golden("lsh_small.npz")
    f = fam(int(g["seed"]))
    for L, K in ((1, 1), (6, 3), (16, 4), (7, 5)):
        res = lsh_batch(g["indptr"], g["ids"], g["w"], LshParams(L, K), f, fps=True)
        assert np.array_equal(as_u64(res.keys), g[f"keys_{L}_{K}"]), (L, K)
        assert np.array_equal(as_u64(res.fps), g[f"fps_{L}_{K}"]), (L, K)


@pytest.mark.parametrize("scale_exp", [None, -200])
def test_lsh_sort_paths_agree(monkeypatch, scale_exp):
    """The fixed-point-key bucket sort and the exact (rank, fp) sort give the
    same keys, also with ||x||_1 = 2^-200 (ranks far beyond the float range:
    the keys are relative to the final limit).  Forced key collisions are
    tested in test_round2.py::test_lsh_fixed_point_key_collisions."""
    indptr, ids, w = workloads.generate("cfg4", n=300, start=777)
    if scale_exp is not None:
        for s in range(indptr.size - 1):
            a, b = indptr[s], indptr[s + 1]
            w[a:b] = np.ldexp(w[a:b] / w[a:b].sum(), scale_exp)
    f = fam(3)
    fast = lsh_batch(indptr, ids, w, LshParams(50, 8), f, fps=True)
    monkeypatch.setenv("DSK_LSH_EXACT", "1")
    exact = lsh_batch(indptr, ids, w, LshParams(50, 8), f, fps=True)
    assert np.array_equal(as_u64(fast.keys), as_u64(exact.keys))
    assert np.array_equal(as_u64(fast.fps), as_u64(exact.fps))
    keys, fps, status, _, _ = Oracle(3).lsh_csr(indptr, ids, w, 50, 8, want_fps=True)
    assert (status == 0).all()
    assert np.array_equal(as_u64(fast.keys), keys)
    assert np.array_equal(as_u64(fast.fps), fps)


def test_minhash_host_multi_device_gather():
    """Single-process multi-GPU host path: row shards through
    dsk_minhash_csr_host written into disjoint slices of the host outputs.
    Three shards on device 0 stand in for three GPUs (same partition logic)."""
    from paper_2005_11547_b200.shard import minhash_host_multi
    indptr, ids, w = workloads.generate("cfg2", n=2000, start=100)
    f = fam(1)
    dev = minhash_batch(indptr, ids, w, 256, f, bits=True)
    for devices in ([0], [0, 0, 0]):
        vals, bits, status = minhash_host_multi(indptr, ids, w, 256, f, devices=devices, bits=True)
        assert (status == 0).all()
        assert np.array_equal(vals, as_u64(dev.values))
        assert np.array_equal(bits, as_u64(dev.bits))


@pytest.mark.parametrize("normalize", [False, True])
def test_lsh_host_multi_device_gather(normalize):
    """The LSH counterpart of minhash_host_multi: row shards through
    dsk_lsh_csr_host into disjoint slices of the host outputs (three shards on
    device 0 stand in for three GPUs), equal to one lsh_batch launch."""
    from paper_2005_11547_b200.shard import lsh_host_multi
    indptr, ids, w = workloads.generate("cfg4", n=1500, start=50)
    f = fam(3)
    prm = LshParams(100, 20)
    dev = lsh_batch(indptr, ids, w, prm, f, normalize=normalize)
    for devices in ([0], [0, 0, 0]):
        keys, status, phi = lsh_host_multi(indptr, ids, w, prm, f, devices=devices,
                                           normalize=normalize)
        assert (status == 0).all()
        assert np.array_equal(keys, as_u64(dev.keys))
        assert np.array_equal(phi, dev.phi.cpu().numpy())


@pytest.mark.parametrize("L,K", [(6000, 1), (5000, 2)])
def test_lsh_large_L_global_counters_vs_oracle(L, K):
    """L beyond the shared-memory bucket counters: counters in global scratch."""
    indptr, ids, w = workloads.generate("cfg1", n=5)
    res = lsh_batch(indptr, ids, w, LshParams(L, K), fam(0), fps=True)
    keys, fps, status, phi, _ = Oracle(0).lsh_csr(indptr, ids, w, L, K, want_fps=True)
    assert (status == 0).all()
    assert np.array_equal(as_u64(res.keys), keys)
    assert np.array_equal(as_u64(res.fps), fps)
    assert np.array_equal(res.phi.cpu().numpy(), phi)


@pytest.mark.parametrize("L,K", [(1, 50), (3, 40), (2, 90)])
def test_lsh_bucket_overflow_list_vs_oracle(monkeypatch, L, K):
    """Buckets past their hit slots (forced to 64) spill into the overflow
    list and are ranked by counting over slots + list."""
    monkeypatch.setenv("DSK_LSH_SLOTS", "64")
    indptr, ids, w = workloads.generate("cfg4", n=60, start=31)
    res = lsh_batch(indptr, ids, w, LshParams(L, K), fam(3), fps=True)
    keys, fps, status, phi, _ = Oracle(3).lsh_csr(indptr, ids, w, L, K, want_fps=True)
    assert (status == 0).all()
    assert np.array_equal(as_u64(res.keys), keys)
    assert np.array_equal(as_u64(res.fps), fps)
    assert np.array_equal(res.phi.cpu().numpy(), phi)


def test_lsh_concurrent_streams():
    """LSH launches on different streams take separate hit-buffer slots."""
    parts = [workloads.generate("cfg4", n=3000, start=s0) for s0 in (0, 3000, 6000, 9000, 12000)]
    f = fam(3)
    serial = [as_u64(lsh_batch(*p, LshParams(100, 20), f).keys) for p in parts]
    dev = torch.device("cuda", 0)
    ins = [tuple(torch.from_numpy(np.asarray(a).view(np.int64) if a.dtype == np.uint64 else a)
                 .to(dev) for a in p) for p in parts]
    streams = [torch.cuda.Stream(dev) for _ in parts]
    torch.cuda.synchronize()
    outs = []
    for st, p in zip(streams, ins):
        with torch.cuda.stream(st):
            outs.append(lsh_batch(*p, LshParams(100, 20), f, check=False))
    torch.cuda.synchronize()
    for o, ref in zip(outs, serial):
        assert np.array_equal(as_u64(o.keys), ref)


def test_lsh_cfg4_vs_oracle():
    indptr, ids, w = workloads.generate("cfg4", n=400, start=5000)
    f = fam(3)
    res = lsh_batch(indptr, ids, w, LshParams(100, 20), f)
    keys, _, status, phi, hits = Oracle(3).lsh_csr(indptr, ids, w, 100, 20)
    assert (status == 0).all()
    assert np.array_equal(as_u64(res.keys), keys)
    assert np.array_equal(res.phi.cpu().numpy(), phi)
    assert np.array_equal(res.stats.cpu().numpy().view(np.uint32)[:, 2].astype(np.int64), hits)
    nres = lsh_batch(indptr, ids, w, LshParams(100, 20), f, normalize=True)
    nkeys, _, nstatus, _, _ = Oracle(3).lsh_csr(indptr, ids, w, 100, 20, normalize=True)
    assert np.array_equal(as_u64(nres.keys), nkeys)


def test_lsh_key_single_set_api():
    f = fam(0xA11)
    x = WeightedSet.from_arrays(np.array([3, 9, 27, 81], dtype=np.uint64),
                                np.array([0.5, 1.5, 0.25, 2.0]))
    keys = lsh_key(x, LshParams(6, 3), f)
    assert len(keys) == 6 and all(len(k) == 3 for k in keys)
    assert keys == lsh_key(x, LshParams(6, 3), f)
    # (L, K) = (1, 1) equals the k = 1 minhash (tests/test_annindex.py:75-78)
    k11 = lsh_key(x, LshParams(1, 1), f)
    assert k11[0][0] == int(dart_minhash(x, 1, f).values[0])
    _, fps, _, _, _ = Oracle(0xA11).lsh_csr(np.array([0, 4]), x.ids, x.weights, 6, 3,
                                             want_fps=True)
    assert [tuple(int(v) for v in row) for row in fps[0]] == keys


def test_darts_random_extreme_weights_vs_oracle():
    """Weight windows under wide dynamic ranges, many t (exercises rho >= 1
    regions and the multiplication-based window estimate)."""
    rng = np.random.default_rng(77)
    f = fam(0x77)
    orc = Oracle(0x77)
    for t in (1, 7, 100, 1000, 5000):
        sets, limits = [], []
        for _ in range(40):
            n = int(rng.integers(1, 30))
            ids = rng.choice(2**40, size=n, replace=False).astype(np.uint64)
            w = 2.0 ** rng.uniform(-40, 40, n)
            l1 = float(np.sum(w))
            limits.append(float(rng.choice([0.5, 1.0, 2.0, 3.0])) / l1)
            sets.append((ids, w))
        indptr = np.zeros(len(sets) + 1, dtype=np.int64)
        np.cumsum([s[0].size for s in sets], out=indptr[1:])
        ids = np.concatenate([s[0] for s in sets])
        w = np.concatenate([s[1] for s in sets])
        offsets, status, cols = darts_batch(indptr, ids, w, t, np.array(limits), f)
        st = status.cpu().numpy()
        off = offsets.cpu().numpy()
        el = as_u64(cols["element"])
        fp = as_u64(cols["fingerprint"])
        rank = cols["rank"].cpu().numpy()
        for s_i in range(len(sets)):
            ost, od = orc.darts_below_rank(sets[s_i][0], sets[s_i][1], t, limits[s_i])
            assert st[s_i] == ost, (t, s_i)
            if ost:
                continue
            a, b = off[s_i], off[s_i + 1]
            got = sorted(zip(el[a:b].tolist(), fp[a:b].tolist(), rank[a:b].tolist()))
            exp = sorted(zip(od["element"].tolist(), od["fingerprint"].tolist(),
                             od["rank"].tolist()))
            assert got == exp, (t, s_i)


def test_lsh_host_buffer_abi():
    import ctypes

    from paper_2005_11547_b200 import _lib
    indptr, ids, w = workloads.generate("cfg4", n=500)
    f = fam(3)
    dev = lsh_batch(indptr, ids, w, LshParams(100, 20), f)
    keys = np.zeros((500, 100), dtype=np.uint64)
    status = np.zeros(500, dtype=np.int32)
    P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    rc = _lib.load().dsk_lsh_csr_host(f.context(), P(indptr), P(ids), P(w), 500, 100, 20, 0,
                                     P(keys), None, P(status), None, None)
    assert rc == 0 and (status == 0).all()
    assert np.array_equal(keys, as_u64(dev.keys))


def test_host_buffer_pinned_and_pageable_mixes():
    """dsk_minhash_csr_host with pinned inputs/outputs (direct DMA), pageable
    ones (staged through the context's pinned buffers) and mixes of both."""
    import ctypes

    from paper_2005_11547_b200 import _lib
    indptr, ids, w = workloads.generate("cfg2", n=3000, start=321)
    f = fam(1)
    ref = as_u64(minhash_batch(indptr, ids, w, 256, f).values)
    P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731

    def pinned(a):
        t = torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).pin_memory()
        out = t.numpy()
        return out.view(np.uint64) if a.dtype == np.uint64 else out

    for pin_in in (False, True):
        for pin_out in (False, True):
            ii = pinned(ids) if pin_in else ids
            ww = pinned(w) if pin_in else w
            vals = pinned(np.zeros((3000, 256), np.uint64)) if pin_out else \
                np.zeros((3000, 256), np.uint64)
            st = pinned(np.zeros(3000, np.int32)) if pin_out else np.zeros(3000, np.int32)
            rc = _lib.load().dsk_minhash_csr_host(f.context(), P(indptr), P(ii), P(ww), 3000, 256,
                                                 P(vals), None, P(st), None, None)
            assert rc == 0 and (st == 0).all()
            assert np.array_equal(vals, ref), (pin_in, pin_out)


@pytest.mark.parametrize("chunk_mb", ["1", "3"])
def test_host_pipeline_many_chunks(monkeypatch, chunk_mb):
    """Small chunk caps: many chunks through the three-stream pipeline (input
    events, kernel events, D2H stream) for both host entry points."""
    import ctypes

    from paper_2005_11547_b200 import _lib
    monkeypatch.setenv("DSK_CHUNK_MB", chunk_mb)
    P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    indptr, ids, w = workloads.generate("cfg3", n=6000)
    f = fam(2)
    dev = minhash_batch(indptr, ids, w, 64, f)
    vals = np.zeros((6000, 64), dtype=np.uint64)
    status = np.full(6000, -1, dtype=np.int32)
    rc = _lib.load().dsk_minhash_csr_host(f.context(), P(indptr), P(ids), P(w), 6000, 64, P(vals),
                                         None, P(status), None, None)
    assert rc == 0 and (status == 0).all()
    assert np.array_equal(vals, as_u64(dev.values))
    # ids wider than 32 bits in the second half of the rows
    wide = ids.copy()
    wide[indptr[3000]:] += np.uint64(1 << 40)
    dev_w = minhash_batch(indptr, wide, w, 64, f)
    vals[:] = 0
    rc = _lib.load().dsk_minhash_csr_host(f.context(), P(indptr), P(wide), P(w), 6000, 64,
                                         P(vals), None, P(status), None, None)
    assert rc == 0 and (status == 0).all()
    assert np.array_equal(vals, as_u64(dev_w.values))
    indptr, ids, w = workloads.generate("cfg4", n=1500)
    dev = lsh_batch(indptr, ids, w, LshParams(30, 4), f, fps=True)
    keys = np.zeros((1500, 30), dtype=np.uint64)
    fps = np.zeros((1500, 30, 4), dtype=np.uint64)
    status = np.full(1500, -1, dtype=np.int32)
    phi = np.zeros(1500, dtype=np.int32)
    rc = _lib.load().dsk_lsh_csr_host(f.context(), P(indptr), P(ids), P(w), 1500, 30, 4, 0,
                                     P(keys), P(fps), P(status), P(phi), None)
    assert rc == 0 and (status == 0).all()
    assert np.array_equal(keys, as_u64(dev.keys))
    assert np.array_equal(fps, as_u64(dev.fps))
    assert np.array_equal(phi, dev.phi.cpu().numpy())


def test_tie_resolution_path():
    """Rows flagged DSK_STATUS_TIE are re-resolved by full index tuple on the
    GPU (ref/sketching.py:93-99); force the path on corrupted rows."""
    from paper_2005_11547_b200 import api
    indptr, ids, w = workloads.generate("cfg1", n=40)
    f = fam(0)
    k = 64
    res = minhash_batch(indptr, ids, w, k, f, bits=True)
    good = as_u64(res.values).copy()
    good_bits = as_u64(res.bits).copy()
    rows = torch.tensor([3, 17, 29], device=res.values.device)
    res.values[rows] = 12345
    res.bits[rows] = 0
    res.status[rows] = res.status[rows] | DSK_STATUS_TIE
    dev = res.values.device
    p = torch.from_numpy(indptr).to(dev)
    i = torch.from_numpy(ids.view(np.int64)).to(dev)
    ww = torch.from_numpy(w).to(dev)
    api._resolve_minhash_ties(res, p, i, ww, k, f, dev)
    assert np.array_equal(as_u64(res.values), good)
    assert np.array_equal(as_u64(res.bits), good_bits)
    assert (res.status.cpu().numpy() == 0).all()


@pytest.mark.parametrize("normalize", [False, True])
def test_lsh_tie_resolution_path(normalize):
    """LSH rows flagged DSK_STATUS_TIE are re-keyed by full index tuple on the
    GPU (ref/annindex.py:77-81, :135); force the path on corrupted rows."""
    from paper_2005_11547_b200 import api
    indptr, ids, w = workloads.generate("cfg4", n=30, start=11)
    f = fam(3)
    params = LshParams(40, 5)
    res = lsh_batch(indptr, ids, w, params, f, fps=True, normalize=normalize)
    good_k, good_f = as_u64(res.keys).copy(), as_u64(res.fps).copy()
    rows = torch.tensor([2, 9, 21], device=res.keys.device)
    res.keys[rows] = 7
    res.fps[rows] = 7
    res.status[rows] = res.status[rows] | DSK_STATUS_TIE
    dev = res.keys.device
    p = torch.from_numpy(indptr).to(dev)
    i = torch.from_numpy(ids.view(np.int64)).to(dev)
    ww = torch.from_numpy(w).to(dev)
    api._resolve_lsh_ties(res, p, i, ww, params, f, dev, normalize)
    assert np.array_equal(as_u64(res.keys), good_k)
    assert np.array_equal(as_u64(res.fps), good_f)
    assert (res.status.cpu().numpy() == 0).all()


# ------------------------------------------------- bottom-k and DSK1 (next rows)


def test_l1_batch_matches_numpy():
    from paper_2005_11547_b200 import l1_batch
    rng = np.random.default_rng(4)
    sizes = [0, 1, 5, 8, 127, 128, 129, 1000, 1024, 4097, 16384, 16385, 40000]
    lens = np.array(sizes, dtype=np.int64)
    indptr = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    w = rng.lognormal(0.0, 3.0, int(indptr[-1]))
    got = l1_batch(indptr, w).cpu().numpy()
    exp = np.array([float(np.sum(w[indptr[s]:indptr[s + 1]])) for s in range(lens.size)])
    assert np.array_equal(got, exp)


def test_bottom_k_golden():
    from paper_2005_11547_b200 import bottom_k_batch
    g = golden("bottomk_dsk1.npz")
    f = fam(int(g["seed"]))
    n = g["indptr"].size - 1
    for k in (1, 3, 17, 64):
        res = bottom_k_batch(g["indptr"], g["ids"], g["w"], k, f)
        exp = g[f"bottomk_k{k}"].reshape(n, k)
        cols = {name: v.cpu().numpy() for name, v in res.columns.items()}
        for name in exp.dtype.names:
            got = cols[name]
            if name in ("element", "fingerprint"):
                got = got.view(np.uint64)
            elif name in ("nu", "rho", "j"):
                got = got.view(np.uint16)
            elif name in ("w", "r"):
                got = got.view(np.uint32)
            assert np.array_equal(got, exp[name]), (k, name)


def test_bottom_k_single_set_api_and_oracle():
    from paper_2005_11547_b200 import bottom_k
    f = fam(0xBEEF)
    x = make_weighted_set([(1, 0.5), (2, 0.25), (3, 1.25)])
    sk = bottom_k(x, 12, f)
    # tests/test_sketching.py:112-117: prefix of the (rank, index)-ordered darts
    universe = DartHasher(12, f).darts(x, 64.0)
    assert sk.darts == sorted(universe, key=lambda d: (d.rank, d.index))[:12]
    indptr, ids, w = workloads.generate("cfg3", n=40)
    orc = Oracle(2)
    from paper_2005_11547_b200 import bottom_k_batch
    res = bottom_k_batch(indptr, ids, w, 64, fam(2))
    fp = as_u64(res.columns["fingerprint"])
    for s in range(40):
        st, _, od = orc.bottom_k(ids[indptr[s]:indptr[s + 1]], w[indptr[s]:indptr[s + 1]], 64)
        assert st == 0 and np.array_equal(fp[s], od["fingerprint"])


def _dart_rows(offsets, cols, q):
    off = offsets.cpu().numpy()
    a, b = off[q], off[q + 1]
    arr = np.empty(b - a, dtype=[("element", "<u8"), ("nu", "<u2"), ("rho", "<u2"),
                                 ("w", "<u4"), ("r", "<u4"), ("j", "<u2"),
                                 ("weight", "<f8"), ("rank", "<f8"), ("fingerprint", "<u8")])
    for name in arr.dtype.names:
        v = cols[name][a:b].cpu().numpy()
        arr[name] = v.view(arr.dtype[name]) if v.dtype.itemsize == arr.dtype[name].itemsize \
            else v
    return arr


def test_darts_and_bottom_k_large_sets_vs_oracle():
    """Sets beyond the row sink's 4096-element slice: enumerated slice by
    slice, darts tuple-for-tuple and bottom-k identical to the oracle."""
    lens = [4095, 4096, 4097, 9000, 1, 20000]
    indptr, ids, w = _ragged_batch(31, lens, sigma=1.5)
    f = fam(0x31)
    orc = Oracle(0x31)
    limits = np.array([1.0 / float(np.sum(w[indptr[s]:indptr[s + 1]])) for s in range(len(lens))])
    offsets, status, cols = darts_batch(indptr, ids, w, 64, limits, f)
    assert (status.cpu().numpy() == 0).all()
    for s in range(len(lens)):
        st, od = orc.darts_below_rank(ids[indptr[s]:indptr[s + 1]], w[indptr[s]:indptr[s + 1]],
                                      64, float(limits[s]))
        assert st == 0
        got = canonical_darts(_dart_rows(offsets, cols, s))
        assert np.array_equal(got, canonical_darts(od)), s
    # area cap over the whole set (ref/darthash.py:242-244) when no single
    # lane's share exceeds it: 20000 elements, ~2.5e8 areas in total
    cid = np.arange(20000, dtype=np.uint64) * 7 + 3
    cw = np.ones(20000)
    _, cst, _ = darts_batch(np.array([0, 20000]), cid, cw, 64, np.array([100.0]), f)
    assert cst.cpu().numpy()[0] == 4 == orc.darts_below_rank(cid, cw, 64, 100.0)[0]
    from paper_2005_11547_b200 import bottom_k_batch
    res = bottom_k_batch(indptr, ids, w, 50, f)
    fp = as_u64(res.columns["fingerprint"])
    rk = res.columns["rank"].cpu().numpy()
    for s in range(len(lens)):
        st, phi, od = orc.bottom_k(ids[indptr[s]:indptr[s + 1]], w[indptr[s]:indptr[s + 1]], 50)
        assert st == 0
        assert np.array_equal(fp[s], od["fingerprint"]), s
        assert np.array_equal(rk[s], od["rank"]), s


def test_bottom_k_fused_spill_and_large_k_paths(monkeypatch):
    """The fused bottom-k kernel, its DSK_SCRATCH fallback (forced with a
    tiny buffer) and the composed path for k > 256 all equal the oracle."""
    from paper_2005_11547_b200 import bottom_k_batch
    indptr, ids, w = workloads.generate("cfg3", n=30, start=900)
    orc = Oracle(2)
    f = fam(2)
    exp = {}
    for k in (64, 200, 256, 300):
        exp[k] = np.stack([orc.bottom_k(ids[indptr[s]:indptr[s + 1]],
                                        w[indptr[s]:indptr[s + 1]], k)[2]["fingerprint"]
                           for s in range(30)])
    for k in (64, 200, 256):
        fused = as_u64(bottom_k_batch(indptr, ids, w, k, f).columns["fingerprint"])
        assert np.array_equal(fused, exp[k]), k
    monkeypatch.setenv("DSK_BOTTOMK_CAP", "40")
    spilled = bottom_k_batch(indptr, ids, w, 64, f)
    assert np.array_equal(as_u64(spilled.columns["fingerprint"]), exp[64])
    assert (spilled.status.cpu().numpy() == 0).all()
    monkeypatch.delenv("DSK_BOTTOMK_CAP")
    big = as_u64(bottom_k_batch(indptr, ids, w, 300, f).columns["fingerprint"])
    assert np.array_equal(big, exp[300])


def test_dsk1_records_byte_identical():
    from paper_2005_11547_b200 import (BottomKFingerprints, MinHashSketch, bottom_k_batch,
                                       dump_sketches, iter_sketches)
    g = golden("bottomk_dsk1.npz")
    f = fam(int(g["seed"]))
    res = minhash_batch(g["indptr"], g["ids"], g["w"], 100, f, bits=True)
    assert dump_sketches(res.values, 1, 100, f.seed) == g["dsk1_minhash"].tobytes()
    assert dump_sketches(res.bits, 2, 100, f.seed) == g["dsk1_onebit"].tobytes()
    bk = bottom_k_batch(g["indptr"], g["ids"], g["w"], 17, f)
    assert dump_sketches(bk.columns["fingerprint"], 3, 17, f.seed) == g["dsk1_bottomk"].tobytes()
    recs = list(iter_sketches(g["dsk1_minhash"].tobytes()))
    assert isinstance(recs[0], MinHashSketch)
    assert np.array_equal(np.stack([r.values for r in recs]), as_u64(res.values))
    assert isinstance(list(iter_sketches(g["dsk1_bottomk"].tobytes()))[0], BottomKFingerprints)
    # word-aligned one-bit records (k = 256: 32-byte payload) against
    # struct.pack + np.packbits as ref/sketching.py:224-231 writes them
    import struct
    r2 = minhash_batch(g["indptr"], g["ids"], g["w"], 256, f, bits=True)
    bits = (as_u64(r2.values) & np.uint64(1)).astype(np.uint8)
    exp = b"".join(struct.pack("<4sBBHIQ", b"DSK1", 1, 2, 0, 256, f.seed) +
                   np.packbits(row, bitorder="little").tobytes() for row in bits)
    assert dump_sketches(r2.bits, 2, 256, f.seed) == exp


# ------------------------------------------------------- LshIndex (next row)


def _sets_from_csr(indptr, ids, w):
    return [WeightedSet.from_arrays(ids[indptr[s]:indptr[s + 1]], w[indptr[s]:indptr[s + 1]])
            for s in range(indptr.size - 1)]


def test_lsh_index_matches_reference():
    from paper_2005_11547_b200 import LshIndex
    g = golden("lsh_index.npz")
    f = fam(int(g["seed"]))
    params = LshParams(int(g["L"]), int(g["K"]), float(g["j1"]))
    idx = LshIndex(params, f, debug=True)
    pts = _sets_from_csr(g["p_indptr"], g["p_ids"], g["p_w"])
    idx.insert_many(list(range(50)), pts[:50])
    for i in range(50, len(pts)):  # single inserts interleaved with a query
        idx.insert(i, pts[i])
    assert len(idx) == len(pts)
    for i in range(len(pts)):
        c, keys = idx._debug_keys[i]
        assert c == g["classes"][i]
        assert np.array_equal(keys, g["keys"][i])
    qs = _sets_from_csr(g["q_indptr"], g["q_ids"], g["q_w"])
    results = idx.query_many(qs)
    ptr = g["res_ptr"]
    for qi, r in enumerate(results):
        exp = list(zip(g["res_pid"][ptr[qi]:ptr[qi + 1]].tolist(),
                       g["res_score"][ptr[qi]:ptr[qi + 1]].tolist()))
        assert r == exp, qi
    assert idx.query(qs[3]) == results[3]


def test_lsh_index_semantics():
    from paper_2005_11547_b200 import LshIndex
    f = fam(0x1E0)
    idx = LshIndex(LshParams(L=4, K=2), f)
    assert idx.query(make_weighted_set([(1, 1.0)])) == []
    rng = np.random.default_rng(4)
    xs = [WeightedSet.from_arrays(rng.choice(10**6, 12, replace=False).astype(np.uint64),
                                  rng.random(12) * 2.0 ** rng.uniform(-3, 3) + 1e-3)
          for _ in range(20)]
    idx.insert_many(range(20), xs)
    for i, x in enumerate(xs):  # tests/test_annindex.py:94-103
        r = idx.query(x)
        assert r and r[0] == (i, 1.0)
    with pytest.raises(ValidationError):
        idx.insert(3, xs[0])
    with pytest.raises(ValidationError):
        idx.insert(99, make_weighted_set([]))
    with pytest.raises(ValidationError):
        idx.query(make_weighted_set([]))


# ------------------------------------------- statistical laws (cheap re-checks)


def _pair(rng, l0, J):
    """x and a companion y with weighted Jaccard J (ref/bench.py:103-121 construction)."""
    ids = rng.choice(2**40, l0, replace=False).astype(np.uint64)
    e = -np.log1p(-rng.random(l0))
    w = e / e.sum()
    b = 2.0 * J / (1.0 + J)
    fresh = np.uint64(2**41 + int(rng.integers(0, 2**20)))
    y_ids = np.concatenate([ids, [fresh]])
    y_w = np.concatenate([w * b, [(1.0 - b) * float(np.sum(w))]])
    return (ids, w), (y_ids, y_w)


def test_collision_rate_tracks_similarity():
    # tests/test_sketching.py:65-76: per coordinate P[collision] = J
    k, trials, J = 256, 200, 0.5
    rng = np.random.default_rng(900)
    rows = []
    for _ in range(trials):
        x, y = _pair(rng, 24, J)
        rows += [x, y]
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum([r[0].size for r in rows], out=indptr[1:])
    ids = np.concatenate([r[0] for r in rows])
    w = np.concatenate([r[1] for r in rows])
    v = as_u64(minhash_batch(indptr, ids, w, k, fam(7000)).values)
    est = (v[0::2] == v[1::2]).mean()
    se = (J * (1 - J) / (k * trials)) ** 0.5
    assert abs(est - J) <= 4 * se


def test_dart_count_is_poisson():
    # tests/test_darthash.py:85-96: mean dart count at phi = 1 is t
    from paper_2005_11547_b200 import l1_batch
    rng = np.random.default_rng(1312)
    t, sets = 1000, 400
    lens = np.full(sets, 32)
    indptr = np.zeros(sets + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    ids = np.concatenate([rng.choice(2**40, 32, replace=False) for _ in range(sets)]).astype(np.uint64)
    w = rng.random(indptr[-1]) + 1e-3
    l1 = l1_batch(indptr, w).cpu().numpy()
    offsets, status, _ = darts_batch(indptr, ids, w, t, 1.0 / l1, fam(11))
    counts = np.diff(offsets.cpu().numpy())
    assert (status.cpu().numpy() == 0).all()
    assert abs(counts.mean() - t) <= 4 * (t / sets) ** 0.5
    assert abs(counts.var() / t - 1.0) < 0.25


# ------------------------------------------------------ ICWS comparator (f4)


@pytest.mark.parametrize("k", [64, 200])
def test_icws_matches_reference(k):
    """ICWS samples and fingerprints against the reference's own outputs
    (ref/baselines.py:84-161): cfg3 rows plus weights over 2^+-30."""
    from paper_2005_11547_b200 import icws_batch, icws_fingerprints, IcwsHashValue
    g = golden("icws.npz")
    f = fam(int(g["seed"]))
    res = icws_batch(g["indptr"], g["ids"], g["w"], k, f)
    el = as_u64(res.element)
    tk = res.tick.cpu().numpy()
    mism = int(((el != g[f"element_k{k}"]) | (tk != g[f"tick_k{k}"])).sum())
    assert mism == 0, f"{mism} of {el.size} samples differ (libm vs libdevice log)"
    vals = [IcwsHashValue(int(e), int(t)) for e, t in zip(el[0], tk[0])]
    assert np.array_equal(icws_fingerprints(vals, f), g[f"fp_k{k}"][0])


def test_icws_api_semantics():
    from paper_2005_11547_b200 import IcwsSketcher, icws_estimate_jaccard, icws_minhash
    f = fam(9)
    x = make_weighted_set([(1, 0.5), (2, 2.0), (7, 1.25)])
    a = icws_minhash(x, 32, f)
    assert a == IcwsSketcher(32, f, fast=True).minhash(x)
    assert icws_estimate_jaccard(a, a) == 1.0
    with pytest.raises(ValidationError):
        icws_minhash(make_weighted_set([]), 8, f)
    with pytest.raises(ValidationError):
        IcwsSketcher(0, f)
