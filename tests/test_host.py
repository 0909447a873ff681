"""CPU-only tests of the host side: the C-ABI library loads and exports every
symbol include/dsk_b200.h declares, the host constants reproduce the
reference's (golden-pinned) values, and the workload generator is
deterministic and shard-independent.  No compute call is made here."""

import math
import os
import re

import numpy as np
import pytest
import torch

from conftest import REPO, golden
from paper_2005_11547_b200 import HashFamily, _lib, constants, workloads


def header_symbols():
    hdr = open(os.path.join(REPO, "include", "dsk_b200.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(dsk_\w+)\s*\(", hdr, flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 14
    for name in syms:
        assert hasattr(lib, name), name
    assert {n for n, _, _ in _lib.SIGNATURES} == set(syms)


def test_minhash_density_host_abi():
    lib = _lib.load()
    for k, t in ((1, 1), (2, 4), (64, 331), (128, 750), (256, 1676), (1024, 8122)):
        assert lib.dsk_minhash_density(k) == t
        assert constants.minhash_density(k) == t
    g = golden("misc.npz")
    for k, d in zip(g["ks"].tolist(), g["density"].tolist()):
        assert lib.dsk_minhash_density(k) == d


def _py_hash64(tab, element, nu, rho, w, r, j, stream):
    import struct
    key = struct.pack("<QBBIIHH", element, nu, rho, w, r, j, stream)
    h = 0
    for p in range(22):
        h ^= int(tab[p, key[p]])
    m = 2**64 - 1
    h ^= h >> 30
    h = (h * 0xBF58476D1CE4E5B9) & m
    h ^= h >> 27
    h = (h * 0x94D049BB133111EB) & m
    return h ^ (h >> 31)


def test_tables_reproduce_golden_hash():
    tab = constants.hash_tables(1)
    assert _py_hash64(tab, 123, 4, 5, 6, 7, 8, 9) == 317886004245365293
    g = golden("hash_vectors.npz")
    tab = constants.hash_tables(int(g["seed"]))
    for i in range(0, 2000, 97):
        for s_idx, s in enumerate(g["streams"].tolist()):
            assert _py_hash64(tab, int(g["elem"][i]), int(g["nu"][i]), int(g["rho"][i]),
                              int(g["w"][i]), int(g["r"][i]), int(g["j"][i]), s) == \
                int(g["out"][s_idx][i])


def test_poisson_cdf_matches_reference():
    g = golden("hash_vectors.npz")
    assert np.array_equal(constants.poisson1_cdf(), g["cdf"])
    cdf = constants.poisson1_cdf()
    thr = np.ceil(np.ldexp(cdf, 53))
    # X >= ceil(cdf*2^53)  <=>  X * 2^-53 >= cdf  for integer X < 2^53
    rng = np.random.default_rng(0)
    X = rng.integers(0, 2**53, 200000, dtype=np.int64)
    for m in range(20):
        t = int(thr[m])
        for x in (t - 1, t, t + 1):
            if 0 <= x < 2**53:
                assert (x >= t) == (x * 2.0**-53 >= cdf[m])
    ref = np.searchsorted(cdf, X * 2.0**-53, side="right")
    got = (X[:, None] >= thr[None, :].astype(np.int64)).sum(1)
    assert np.array_equal(ref, got)


def test_log2_threshold_depth_formula():
    f = constants.floor_log2_via_thresholds
    rng = np.random.default_rng(1)
    ys = list(2.0 ** rng.uniform(0, 255, 20000)) + [1.0, 2.0, 3.0, 4.0]
    for n in range(1, 257):
        p = math.ldexp(1.0, n)
        y = p
        for _ in range(400):
            y = math.nextafter(y, 0.0)
            ys.append(y)
        y = p
        for _ in range(3):
            ys.append(y)
            y = math.nextafter(y, math.inf)
    for y in ys:
        if y >= 1.0 and math.log2(y) < 256:
            assert f(y) == math.floor(math.log2(y)), y


def test_workloads_deterministic_and_shardable():
    a = workloads.generate("cfg3", n=300)
    b = workloads.generate("cfg3", n=300)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    p, i, w = workloads.generate("cfg3", n=100, start=150)
    assert np.array_equal(p, a[0][150:251] - a[0][150])
    assert np.array_equal(i, a[1][a[0][150]:a[0][250]])
    for r in range(300):
        seg = a[1][a[0][r]:a[0][r + 1]]
        assert np.unique(seg).size == seg.size
    p5, i5, w5 = workloads.generate("cfg5", n=2000)
    nnz = np.diff(p5)
    assert nnz.min() >= 1 and nnz.max() <= 16384 and np.median(nnz) <= 3
    p2, _, w2 = workloads.generate("cfg2", n=20)
    sums = np.add.reduceat(w2, p2[:-1])
    assert np.allclose(sums, 1.0)


def test_no_cpu_path_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    f = HashFamily(1)
    with pytest.raises(RuntimeError, match="CUDA"):
        f.hash64(1)


def test_bench_reference_arm_json_contract():
    """`bench.py --impl reference` runs on the host alone and prints the
    contract's JSON line (impl, metric, cpu_baseline, zero-copy e2e)."""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--impl", "reference",
                          "--workload", "cfg1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, check=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert key in line, key
    assert line["impl"] == "reference" and line["metric"] == "sketches/sec"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_shape_hint_withheld_for_mostly_small_batches():
    """dsk_minhash_csr_ex's team-shape hint (results never depend on it): the
    batch's nonzeros for uniform large sets, 0 when half of the sampled rows
    hold < 48 elements (cfg5's Zipf sizes run faster on single-warp teams)."""
    import torch
    from paper_2005_11547_b200.api import _shape_hint
    from paper_2005_11547_b200 import workloads
    for name, want_zero in (("cfg2", False), ("cfg5", True)):
        indptr, ids, _ = workloads.generate(name, n=5000)
        p = torch.from_numpy(indptr)
        i = torch.from_numpy(ids.view(np.int64))
        hint_host = _shape_hint(indptr, p, i)
        # tensor inputs are sampled on the device by dsk_minhash_hints (GPU test:
        # test_minhash_direct_first_handoff checks both samples agree)
        assert _shape_hint(p, p, i) == -1
        assert (hint_host == 0) == want_zero
        if not want_zero:
            assert hint_host == int(indptr[-1])
    # direct-first bit: raw cfg3 weights (l1 ~ 32) qualify, cfg2's normalised ones do not
    from paper_2005_11547_b200.api import HINT_DIRECT
    for name, want in (("cfg3", True), ("cfg2", False)):
        indptr, ids, w = workloads.generate(name, n=5000)
        p = torch.from_numpy(indptr)
        i = torch.from_numpy(ids.view(np.int64))
        assert bool(_shape_hint(indptr, p, i, w) & HINT_DIRECT) == want
