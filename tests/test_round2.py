"""Fidelity checks added in round 2: OverflowError depths, duplicate ids,
the set-file reader and the GPU `sketch` command, the reference names the
facade mirrors (DartBatch.empty/take, exact_jaccard, derive_seed), tie repair
on the host-buffer path, and the shard plan from row lengths."""

from __future__ import annotations

import math
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO, golden

from oracle.oracle import Oracle
from paper_2005_11547_b200 import (DartBatch, ValidationError, derive_seed, shard, workloads)
from paper_2005_11547_b200 import io as dio


# ----------------------------------------------------------------- CPU side

def test_derive_seed_known_answer():
    # the reference's derive_seed(1, 2, 3) (ref/randomness.py:89-92), run in the build container
    assert derive_seed(1, 2, 3) == 10928566898365450891
    assert workloads.derive_seed is derive_seed


def test_dartbatch_empty_and_take():
    e = DartBatch.empty()
    assert e.size == 0
    assert [getattr(e, n).dtype for n in DartBatch.__slots__] == [
        np.uint64, np.uint16, np.uint16, np.uint32, np.uint32, np.uint16, np.float64, np.float64,
        np.uint64]
    cols = [np.arange(5, dtype=getattr(e, n).dtype) + i for i, n in enumerate(DartBatch.__slots__)]
    b = DartBatch(*cols).take(np.array([4, 1]))
    assert b.size == 2
    for i, n in enumerate(DartBatch.__slots__):
        assert getattr(b, n).tolist() == [4 + i, 1 + i]


def test_oracle_overflow_statuses():
    """The C oracle maps 1 + t*x = inf to OverflowError (status 9), a finite
    depth > 255 to ValidationError (3) and l1 = inf to the limit error (6),
    as the reference does (tests/golden/overflow.npz, made by the reference)."""
    g = golden("overflow.npz")
    orc = Oracle(int(g["seed"]))
    for k in (1, 64):
        _, status, _, _ = orc.minhash_csr(g["indptr"], g["ids"], g["w"], k)
        assert status.tolist() == g[f"status_k{k}"].tolist()
    _, _, status, _, _ = orc.lsh_csr(g["indptr"], g["ids"], g["w"], 4, 2)
    assert status.tolist() == g["status_lsh"].tolist()


def _cli_golden_text():
    g = golden("cli_sketch.npz")
    return g, g["text"].tobytes().decode()


def test_read_csr_matches_the_reference_text(tmp_path):
    """read_csr drops blank lines and zero weights; writing the CSR back gives
    the reference's format_set text of every kept pair."""
    g, text = _cli_golden_text()
    path = tmp_path / "sets.txt"
    path.write_text(text)
    indptr, ids, w = dio.read_csr(path)
    expect = []
    for line in text.split("\n"):
        if not line.strip():
            continue
        toks = [t for t in line.split() if float(t.partition(":")[2]) != 0.0]
        expect.append(" ".join(toks))
    assert indptr.size - 1 == len(expect)
    out = tmp_path / "back.txt"
    dio.write_csr(out, indptr, ids, w)
    assert out.read_text() == "\n".join(expect) + "\n"
    sets = dio.read_sets(path)
    assert [x.l0 for x in sets] == np.diff(indptr).tolist()
    assert all(x.l1 == float(np.sum(x.weights)) for x in sets)


@pytest.mark.parametrize("name", ["neg_then_malformed", "malformed", "dup", "range", "nonfinite",
                                  "inf"])
def test_cli_parse_errors_match_the_reference(tmp_path, name):
    """Bad set files: same exit code and stderr as `dartsketch sketch`
    (ref/cli.py:107-131, ref/core.py:69-100), before any GPU work."""
    g = golden("cli_sketch.npz")
    path = tmp_path / f"{name}.txt"
    path.write_bytes(g[f"badtext_{name}"].tobytes())
    proc = subprocess.run([sys.executable, "-m", "paper_2005_11547_b200.cli", "sketch",
                           "--input", str(path), "--out", str(tmp_path / "o.dsk")],
                          cwd=REPO, capture_output=True, text=True, timeout=300)
    assert proc.returncode == int(g[f"badrc_{name}"])
    assert proc.stderr.replace(str(path), "<path>") == str(g[f"baderr_{name}"])


def test_plan_shards_lengths_matches_plan_shards():
    lens = workloads.lengths("cfg5", 50000, start=1234)
    indptr = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    for world in (1, 2, 3, 8):
        a = shard.plan_shards(indptr, world, 750)
        b = shard.plan_shards_lengths(lens, world, 750)
        assert np.array_equal(a, b)
        assert a[0] == 0 and a[-1] == lens.size and (np.diff(a) >= 0).all()


def test_generate_is_independent_of_workers_and_split():
    """Rows come out identical whatever the worker count and row range."""
    a = workloads.generate("cfg5", n=70000, start=60000, workers=1)
    b = workloads.generate("cfg5", n=70000, start=60000, workers=4)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    p, i, w = workloads.generate("cfg5", n=30000, start=90000, workers=2)
    lo, hi = a[0][30000], a[0][60000]
    assert np.array_equal(p, a[0][30000:60001] - lo)
    assert np.array_equal(i, a[1][lo:hi]) and np.array_equal(w, a[2][lo:hi])
    assert np.array_equal(np.diff(a[0]), workloads.lengths("cfg5", 70000, start=60000))


# ----------------------------------------------------------------- GPU side

@pytest.mark.gpu
def test_overflow_statuses_and_exceptions():
    from paper_2005_11547_b200 import HashFamily, LshParams, lsh_batch, minhash_batch
    g = golden("overflow.npz")
    f = HashFamily(int(g["seed"]))
    for k in (1, 64):
        res = minhash_batch(g["indptr"], g["ids"], g["w"], k, f, check=False)
        assert (res.status.cpu().numpy() & 0xFF).tolist() == g[f"status_k{k}"].tolist()
    res = lsh_batch(g["indptr"], g["ids"], g["w"], LshParams(4, 2), f, check=False)
    assert (res.status.cpu().numpy() & 0xFF).tolist() == g["status_lsh"].tolist()
    # the first row raises what the reference raises: OverflowError at k = 64
    with pytest.raises(OverflowError):
        minhash_batch(g["indptr"][:2], g["ids"][:1], g["w"][:1], 64, f)
    with pytest.raises(ValidationError, match="norm range"):
        minhash_batch(g["indptr"][:2], g["ids"][:1], g["w"][:1], 1, f)


@pytest.mark.gpu
def test_duplicate_ids_rejected_in_row_order():
    from paper_2005_11547_b200 import HashFamily, LshParams, lsh_batch, minhash_batch
    indptr = np.array([0, 2, 4, 5, 7], dtype=np.int64)
    ids = np.array([1, 2, 3, 4, 0, 9, 9], dtype=np.uint64)
    w = np.array([0.5, 0.25, 1.0, 2.0, 0.0, 1.0, 2.0])  # row 2: bad weight; row 3: dup
    f = HashFamily(1)
    with pytest.raises(ValidationError, match="set 2: weights must be finite"):
        minhash_batch(indptr, ids, w, 8, f)
    w[4] = 1.0
    with pytest.raises(ValidationError, match="set 3: duplicate element id"):
        minhash_batch(indptr, ids, w, 8, f)
    with pytest.raises(ValidationError, match="set 3: duplicate element id"):
        lsh_batch(indptr, ids, w, LshParams(4, 2), f)
    res = minhash_batch(indptr, ids, w, 8, f, check=False)  # unchecked: rows run as given
    assert res.values.shape == (4, 8)


@pytest.mark.gpu
def test_exact_jaccard_matches_the_reference_loop():
    from paper_2005_11547_b200 import WeightedSet, exact_jaccard
    rng = np.random.default_rng(5)
    for _ in range(20):
        a = rng.choice(200, size=int(rng.integers(0, 60)), replace=False).astype(np.uint64)
        b = np.concatenate([a[:len(a) // 2],
                            rng.choice(np.arange(200, 400), size=int(rng.integers(1, 40)),
                                       replace=False)]).astype(np.uint64)
        x = WeightedSet.from_arrays(a, rng.random(a.size) + 1e-3)
        y = WeightedSet.from_arrays(b, rng.random(b.size) + 1e-3)
        xm = dict(zip(x.ids.tolist(), x.weights.tolist()))
        ym = dict(zip(y.ids.tolist(), y.weights.tolist()))
        mn = mx = 0.0
        for e in sorted(xm.keys() | ym.keys()):  # ref/core.py:111-119
            mn += min(xm.get(e, 0.0), ym.get(e, 0.0))
            mx += max(xm.get(e, 0.0), ym.get(e, 0.0))
        assert exact_jaccard(x, y) == mn / mx
        assert exact_jaccard(y, x) == mn / mx
    e = WeightedSet.from_arrays(np.zeros(0, np.uint64), np.zeros(0))
    with pytest.raises(ValidationError):
        exact_jaccard(e, e)


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["dartminhash", "icws", "icws-fast", "bottomk"])
@pytest.mark.parametrize("one_bit", [False, True])
def test_cli_sketch_byte_identical(tmp_path, algo, one_bit):
    """`cli sketch` writes the same DSK1 bytes (and errors) as the reference's
    `dartsketch sketch` on the same set file (tests/golden/cli_sketch.npz)."""
    g, text = _cli_golden_text()
    src = tmp_path / "sets.txt"
    src.write_text(text)
    dst = tmp_path / "out.dsk"
    tag = f"{algo.replace('-', '_')}_{'onebit' if one_bit else 'full'}"
    proc = subprocess.run([sys.executable, "-m", "paper_2005_11547_b200.cli", "sketch",
                           "--input", str(src), "--out", str(dst), "--algo", algo, "--k", "64",
                           "--seed", "7"] + (["--one-bit"] if one_bit else []),
                          cwd=REPO, capture_output=True, text=True, timeout=600)
    assert proc.returncode == int(g[f"rc_{tag}"]), proc.stderr
    assert proc.stderr == str(g[f"err_{tag}"])
    if proc.returncode == 0:
        assert dst.read_bytes() == g[f"out_{tag}"].tobytes()


@pytest.mark.gpu
def test_cli_empty_set_error(tmp_path):
    g = golden("cli_sketch.npz")
    path = tmp_path / "e.txt"
    path.write_bytes(g["badtext_empty_set"].tobytes())
    proc = subprocess.run([sys.executable, "-m", "paper_2005_11547_b200.cli", "sketch",
                           "--input", str(path), "--out", str(tmp_path / "o.dsk")],
                          cwd=REPO, capture_output=True, text=True, timeout=300)
    assert proc.returncode == int(g["badrc_empty_set"])
    assert proc.stderr == str(g["baderr_empty_set"])


@pytest.mark.gpu
def test_host_multi_repairs_tied_rows():
    """minhash_host_multi re-resolves DSK_STATUS_TIE rows by index tuple (the
    C entry points leave them fingerprint-ordered): force the repair on
    corrupted rows and get the reference's values and bits back."""
    from paper_2005_11547_b200 import DSK_STATUS_TIE, HashFamily, as_u64, minhash_batch
    from paper_2005_11547_b200.shard import minhash_host_multi, repair_tied_rows
    indptr, ids, w = workloads.generate("cfg1", n=50)
    f = HashFamily(0)
    vals, bits, status = minhash_host_multi(indptr, ids, w, 64, f, devices=[0], bits=True)
    good = minhash_batch(indptr, ids, w, 64, f, bits=True)
    assert np.array_equal(vals, as_u64(good.values)) and np.array_equal(bits, as_u64(good.bits))
    rows = [4, 20, 41]
    vals[rows] = 7
    bits[rows] = 0
    status[rows] |= DSK_STATUS_TIE
    assert repair_tied_rows(indptr, ids, w, 64, f, vals, bits, status) == 3
    assert np.array_equal(vals, as_u64(good.values)) and np.array_equal(bits, as_u64(good.bits))
    assert (status == 0).all()


@pytest.mark.gpu
def test_bits_only_tie_resolution():
    """With values=False the tie path rebuilds the packed words of tied rows
    from the re-resolved minima."""
    import torch

    from paper_2005_11547_b200 import DSK_STATUS_TIE, HashFamily, api, as_u64, minhash_batch
    indptr, ids, w = workloads.generate("cfg3", n=30)
    f = HashFamily(2)
    good = as_u64(minhash_batch(indptr, ids, w, 256, f, bits=True).bits).copy()
    res = minhash_batch(indptr, ids, w, 256, f, values=False, bits=True)
    rows = torch.tensor([2, 11], device=res.bits.device)
    res.bits[rows] = 0
    res.status[rows] |= DSK_STATUS_TIE
    dev = res.bits.device
    p = torch.from_numpy(indptr).to(dev)
    i = torch.from_numpy(ids.view(np.int64)).to(dev)
    ww = torch.from_numpy(w).to(dev)
    api._resolve_minhash_ties(res, p, i, ww, 256, f, dev)
    assert np.array_equal(as_u64(res.bits), good)
    assert (res.status.cpu().numpy() == 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["phi0=1", "phi0=2", "retry"])
@pytest.mark.parametrize("L,K", [(100, 20), (8, 1), (2, 3)])
def test_lsh_first_band_schedules(monkeypatch, mode, L, K):
    """The LSH kernel's first band (0, phi0 / l1] (phi0 = 2 for L >= 8), its
    phi* = 1 recovery, and the retry launch from phi = 1 all give the
    oracle's keys, fingerprints, phi* and H(phi*) (ref/annindex.py:64-82)."""
    from paper_2005_11547_b200 import HashFamily, LshParams, as_u64, lsh_batch
    if mode == "phi0=1":
        monkeypatch.setenv("DSK_LSH_PHI0", "1")
    elif mode == "phi0=2":
        monkeypatch.setenv("DSK_LSH_PHI0", "2")
    else:
        monkeypatch.setenv("DSK_LSH_PHI0", "2")
        monkeypatch.setenv("DSK_LSH_FORCE_RETRY", "1")
    indptr, ids, w = workloads.generate("cfg4", n=400, start=3000)
    res = lsh_batch(indptr, ids, w, LshParams(L, K), HashFamily(3), fps=True)
    keys, fps, status, phi, hits = Oracle(3).lsh_csr(indptr, ids, w, L, K, want_fps=True)
    assert (status == 0).all() and (res.status.cpu().numpy() == 0).all()
    assert np.array_equal(as_u64(res.keys), keys)
    assert np.array_equal(as_u64(res.fps), fps)
    assert np.array_equal(res.phi.cpu().numpy(), phi)
    assert np.array_equal(res.stats.cpu().numpy()[:, 2], hits)
    if (L, K) == (2, 3):
        assert (phi == 1).any()  # the phi* = 1 recovery is exercised


@pytest.mark.gpu
def test_l1_pairwise_all_small_and_deep_sizes():
    """The register-stack numpy pairwise sum (warp_np_sum) equals np.sum for
    every length 0..300, random lengths up to 7e4 and a 2^20 + 13 row (a
    deep recursion), with weights spread over 2^+-20."""
    from paper_2005_11547_b200 import l1_batch
    rng = np.random.default_rng(11)
    sizes = list(range(0, 301)) + rng.integers(301, 70000, 40).tolist() + [2**20 + 13]
    lens = np.array(sizes, dtype=np.int64)
    indptr = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    w = rng.lognormal(0.0, 7.0, int(indptr[-1]))
    got = l1_batch(indptr, w).cpu().numpy()
    exp = np.array([float(np.sum(w[indptr[s]:indptr[s + 1]])) for s in range(lens.size)])
    assert np.array_equal(got, exp)


@pytest.mark.gpu
@pytest.mark.parametrize("qshift", [14, 20, 26])
@pytest.mark.parametrize("L,K", [(100, 20), (2, 3)])
def test_lsh_fixed_point_key_collisions(monkeypatch, qshift, L, K):
    """The K <= 32 selection sorts 32-bit keys {26-bit fixed-point rank, entry
    index}; equal fixed-point ranks among the first K + 1 send the bucket to
    the exact (rank bits, fp) sort.  Coarser keys (DSK_LSH_QSHIFT drops low
    bits: 26 leaves none) force that fallback on some or every bucket; keys,
    fingerprints, phi* (incl. the phi* = 1 recovery of (2, 3)) and H(phi*)
    still equal the oracle's (ref/annindex.py:64-82)."""
    from paper_2005_11547_b200 import HashFamily, LshParams, as_u64, lsh_batch
    monkeypatch.setenv("DSK_LSH_QSHIFT", str(qshift))
    monkeypatch.setenv("DSK_LSH_PHI0", "2")
    indptr, ids, w = workloads.generate("cfg4", n=300, start=4321)
    res = lsh_batch(indptr, ids, w, LshParams(L, K), HashFamily(3), fps=True)
    keys, fps, status, phi, hits = Oracle(3).lsh_csr(indptr, ids, w, L, K, want_fps=True)
    assert (status == 0).all() and (res.status.cpu().numpy() == 0).all()
    assert np.array_equal(as_u64(res.keys), keys)
    assert np.array_equal(as_u64(res.fps), fps)
    assert np.array_equal(res.phi.cpu().numpy(), phi)
    assert np.array_equal(res.stats.cpu().numpy()[:, 2], hits)


@pytest.mark.gpu
@pytest.mark.parametrize("L,K", [(3, 700), (2, 1600)])
def test_lsh_large_K_selection_staging(L, K):
    """Large K: the selected fingerprints of one table fill the team's staged
    rows in shared memory one table at a time (3, 700), or do not fit there
    and go through the global selection buffer (2, 1600); buckets of > 64
    entries take the counting rank.  Keys and fingerprints equal the oracle's."""
    from paper_2005_11547_b200 import HashFamily, LshParams, as_u64, lsh_batch
    indptr, ids, w = workloads.generate("cfg4", n=24, start=99)
    res = lsh_batch(indptr, ids, w, LshParams(L, K), HashFamily(3), fps=True)
    keys, fps, status, phi, hits = Oracle(3).lsh_csr(indptr, ids, w, L, K, want_fps=True)
    assert (status == 0).all() and (res.status.cpu().numpy() == 0).all()
    assert np.array_equal(as_u64(res.keys), keys)
    assert np.array_equal(as_u64(res.fps), fps)
    assert np.array_equal(res.phi.cpu().numpy(), phi)


@pytest.mark.gpu
def test_concurrent_host_calls_on_separate_contexts():
    """Three dsk_minhash_csr_host calls from three host threads, each on its
    own context (as shard.minhash_host_multi drives one context per GPU; here
    all on device 0), with pageable inputs so the host staging threads are
    shared between the concurrent calls: the disjoint output slices equal one
    device launch over the whole batch."""
    import ctypes
    from concurrent.futures import ThreadPoolExecutor

    import torch
    from paper_2005_11547_b200 import HashFamily, _lib, as_u64, constants, minhash_batch
    indptr, ids, w = workloads.generate("cfg2", n=3000, start=500)
    f = HashFamily(1)
    ref = minhash_batch(indptr, ids, w, 256, f, bits=True)
    lib = _lib.load()
    thr = constants.log2_thresholds()
    ctxs = []
    for _ in range(3):
        out = ctypes.c_void_p()
        _lib.check(lib.dsk_ctx_create(0, f._tables.ctypes.data, f.poisson_cdf.ctypes.data,
                                      thr.ctypes.data, ctypes.byref(out)), "dsk_ctx_create")
        ctxs.append(out)
    n, k = indptr.size - 1, 256
    values = np.zeros((n, k), dtype=np.uint64)
    bits = np.zeros((n, 4), dtype=np.uint64)
    status = np.zeros(n, dtype=np.int32)
    bounds = [0, 1000, 2000, n]
    P = ctypes.c_void_p

    def run(r):
        r0, r1 = bounds[r], bounds[r + 1]
        e0 = int(indptr[r0])
        local = np.ascontiguousarray(indptr[r0:r1 + 1] - e0)
        with torch.cuda.device(0):
            return lib.dsk_minhash_csr_host(
                ctxs[r], P(local.ctypes.data), P(ids.ctypes.data + 8 * e0),
                P(w.ctypes.data + 8 * e0), r1 - r0, k, P(values.ctypes.data + 8 * k * r0),
                P(bits.ctypes.data + 8 * 4 * r0), P(status.ctypes.data + 4 * r0), None, None)

    try:
        with ThreadPoolExecutor(max_workers=3) as pool:
            rcs = list(pool.map(run, range(3)))
    finally:
        for c in ctxs:
            lib.dsk_ctx_destroy(c)
    assert rcs == [0, 0, 0]
    assert (status == 0).all()
    assert np.array_equal(values, as_u64(ref.values))
    assert np.array_equal(bits, as_u64(ref.bits))


@pytest.mark.gpu
def test_lsh_direct_engine_and_handoff(monkeypatch):
    """The LSH first launch runs the direct-only engine specialisation (rank
    depth 0); sets whose band needs the region stages (here every other row
    rescaled to ||x||_1 in [1, 2): limit 2 / l1 > 1, rank depth 1) are handed
    to the general-engine retry launch.  Keys, fingerprints, phi* and H(phi*)
    equal the oracle's and the general-engine-only run (DSK_LSH_DIRECT=0)."""
    from paper_2005_11547_b200 import HashFamily, LshParams, as_u64, lsh_batch
    indptr, ids, w = workloads.generate("cfg4", n=400, start=8000)
    w = w.copy()
    for s in range(0, indptr.size - 1, 2):
        a, b = indptr[s], indptr[s + 1]
        w[a:b] = w[a:b] / w[a:b].sum() * 1.5
    f = HashFamily(3)
    res = lsh_batch(indptr, ids, w, LshParams(100, 20), f, fps=True)
    keys, fps, status, phi, hits = Oracle(3).lsh_csr(indptr, ids, w, 100, 20, want_fps=True)
    assert (status == 0).all() and (res.status.cpu().numpy() == 0).all()
    assert np.array_equal(as_u64(res.keys), keys)
    assert np.array_equal(as_u64(res.fps), fps)
    assert np.array_equal(res.phi.cpu().numpy(), phi)
    assert np.array_equal(res.stats.cpu().numpy()[:, 2], hits)
    monkeypatch.setenv("DSK_LSH_DIRECT", "0")
    gen = lsh_batch(indptr, ids, w, LshParams(100, 20), f, fps=True)
    assert np.array_equal(as_u64(gen.keys), keys)
    assert np.array_equal(gen.stats.cpu().numpy(), res.stats.cpu().numpy())


@pytest.mark.gpu
def test_minhash_direct_first_handoff(monkeypatch):
    """Direct-first minhash (DSK_HINT_DIRECT): the direct-only launch sketches
    the sets whose bands have rank depth 0 and hands the others (here every
    third row, rescaled to l1 = 1 so that limit = phi / l1 >= 1) to the
    general launch; values, bits, phi* and H(phi*) equal the plain path's and
    the oracle's, whatever the hint."""
    import torch
    from paper_2005_11547_b200 import HashFamily, _lib, as_u64, minhash_batch
    n, k = 20000, 64
    indptr, ids, w = workloads.generate("cfg3", n=n, start=777)
    w = w.copy()
    for r in range(0, n, 3):
        seg = slice(int(indptr[r]), int(indptr[r + 1]))
        w[seg] /= w[seg].sum()
    f = HashFamily(2)
    monkeypatch.setenv("DSK_MH_DIRECT", "0")
    plain = minhash_batch(indptr, ids, w, k, f, bits=True)
    lib = _lib.load()
    monkeypatch.setenv("DSK_MH_DIRECT", "1")
    l0 = lib.dsk_launch_count()
    res = minhash_batch(indptr, ids, w, k, f, bits=True)
    torch.cuda.synchronize()
    assert lib.dsk_launch_count() - l0 >= 2  # the direct-only launch + the general one
    assert (res.status.cpu().numpy() == 0).all()
    for a, b in ((res.values, plain.values), (res.bits, plain.bits), (res.phi, plain.phi),
                 (res.stats[:, 2:], plain.stats[:, 2:])):
        assert torch.equal(a, b)
    rows = np.arange(0, n, 97)
    sp, si, sw = workloads.subset(indptr, ids, w, rows)
    vals, status, phi, _ = Oracle(2).minhash_csr(sp, si, sw, k)
    assert (status == 0).all()
    assert np.array_equal(as_u64(res.values)[rows], vals)
    assert np.array_equal(res.phi.cpu().numpy()[rows], phi)
    # the facade's own hint: raw cfg3 weights qualify, this mixed batch (a third
    # of the rows normalised) does not
    from paper_2005_11547_b200.api import HINT_DIRECT, _batch_hint
    monkeypatch.delenv("DSK_MH_DIRECT")
    dev = torch.device("cuda", 0)

    def on_dev(*arrs):
        return [torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).to(dev)
                for a in arrs]
    p0, i0, w0 = workloads.generate("cfg3", n=8000)
    tp, ti, tw = on_dev(p0, i0, w0)
    assert _batch_hint(p0, tp, ti, w0, tw, f, dev) == (i0.size | HINT_DIRECT)  # host sample
    assert _batch_hint(tp, tp, ti, tw, tw, f, dev) == (i0.size | HINT_DIRECT)  # device sample
    tp, ti, tw = on_dev(indptr, ids, w)
    assert _batch_hint(indptr, tp, ti, w, tw, f, dev) == ids.size
    assert _batch_hint(tp, tp, ti, tw, tw, f, dev) == ids.size
    # mostly-small rows: no team-shape hint either
    p5, i5, w5 = workloads.generate("cfg5", n=8000)
    tp, ti, tw = on_dev(p5, i5, w5)
    assert _batch_hint(tp, tp, ti, tw, tw, f, dev) & ~HINT_DIRECT == 0
    assert _batch_hint(p5, tp, ti, w5, tw, f, dev) == _batch_hint(tp, tp, ti, tw, tw, f, dev)


@pytest.mark.gpu
def test_minhash_size_split_equals_plain(monkeypatch):
    """Size split of single-warp-team launches (DSK_MH_SPLIT): the rows of
    >= 1024 elements (head of the largest-first order) go to a wide-team
    launch, the rest to the single-warp launch; outputs equal the unsplit
    launch's and the oracle's on the largest rows."""
    import torch
    from paper_2005_11547_b200 import HashFamily, _lib, as_u64, minhash_batch
    n, k = 30000, 128
    indptr, ids, w = workloads.generate("cfg5", n=n, start=4242)
    assert int(np.diff(indptr).max()) >= 4096  # the batch holds large sets
    f = HashFamily(4)
    lib = _lib.load()
    outs, launches = [], []
    monkeypatch.setenv("DSK_MH_DIRECT", "0")  # (a direct-first launch takes no size split)
    for env in ("0", "1"):
        monkeypatch.setenv("DSK_MH_SPLIT", env)
        l0 = lib.dsk_launch_count()
        r = minhash_batch(indptr, ids, w, k, f, bits=True)
        torch.cuda.synchronize()
        launches.append(lib.dsk_launch_count() - l0)
        outs.append(r)
    assert launches[1] == launches[0] + 1  # the wide-team launch
    for a, b in ((outs[0].values, outs[1].values), (outs[0].bits, outs[1].bits),
                 (outs[0].phi, outs[1].phi), (outs[0].stats[:, 2:], outs[1].stats[:, 2:])):
        assert torch.equal(a, b)
    rows = np.argsort(np.diff(indptr))[-12:]
    sp, si, sw = workloads.subset(indptr, ids, w, rows)
    vals, status, phi, _ = Oracle(4).minhash_csr(sp, si, sw, k)
    assert (status == 0).all()
    assert np.array_equal(as_u64(outs[1].values)[rows], vals)
    assert np.array_equal(outs[1].phi.cpu().numpy()[rows], phi)
