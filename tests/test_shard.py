"""Multi-process (gloo, world_size 2, CPU) tests of the row-sharding host
logic: shard planning, local CSR slicing and the optional result gather.
The GPU compute is stood in for by a row-id function so the test checks that
every row lands exactly once and in order."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_11547_b200 import shard, workloads


def test_plan_shards_balanced_and_complete():
    indptr, _, _ = workloads.generate("cfg5", n=20000)
    for world in (1, 2, 3, 4, 8):
        b = shard.plan_shards(indptr, world, t=750)
        assert b[0] == 0 and b[-1] == 20000 and (np.diff(b) >= 0).all()
        cost = shard.row_costs(indptr, 750)
        per = np.array([cost[b[r]:b[r + 1]].sum() for r in range(world)])
        assert per.max() <= cost.sum() / world + cost.max() + 1e-9


def test_shard_csr_slices():
    indptr, ids, w = workloads.generate("cfg3", n=1000)
    b = shard.plan_shards(indptr, 3, t=331)
    got_ids, got_w, rows = [], [], 0
    for r in range(3):
        p, i, ww = shard.shard_csr(indptr, ids, w, b, r)
        assert p[0] == 0 and p[-1] == i.size == ww.size
        rows += p.size - 1
        got_ids.append(i)
        got_w.append(ww)
    assert rows == 1000
    assert np.array_equal(np.concatenate(got_ids), ids)
    assert np.array_equal(np.concatenate(got_w), w)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    indptr, _, _ = workloads.generate("cfg5", n=3001)
    bounds = shard.plan_shards(indptr, world, t=750)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    # stand-in for the per-rank GPU result: one row of 4 values per set
    local = torch.arange(r0, r1, dtype=torch.int64).unsqueeze(1).repeat(1, 4) * 10 + rank
    full = shard.gather_rows(local, bounds)
    ok = full.shape == (3001, 4) and bool((full[:, 0] // 10 == torch.arange(3001)).all())
    owners = (full[:, 0] % 10).numpy()
    exp = np.concatenate([np.full(int(bounds[r + 1] - bounds[r]), r) for r in range(world)])
    ok = ok and np.array_equal(owners, exp)
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gather_rows_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def _rank_rows_worker(rank, world, port, q, use_gpu):
    """bench.py's strong-scaling data path: plan from row lengths alone, each
    rank generates only its own rows; with use_gpu the rows are sketched on
    the (shared) GPU and the outputs gathered over gloo."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 20000
    lens = workloads.lengths("cfg5", n)
    bounds = shard.plan_shards_lengths(lens, world, 750)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    p, i, w = workloads.generate("cfg5", n=r1 - r0, start=r0, workers=2)
    if use_gpu:
        from paper_2005_11547_b200 import HashFamily, minhash_batch
        res = minhash_batch(p, i, w, 128, HashFamily(4), bits=True, device="cuda:0")
        local = torch.cat([res.values, res.bits, res.status.to(torch.int64).unsqueeze(1)],
                          dim=1).cpu()
    else:
        local = torch.from_numpy(np.stack([np.diff(p), np.add.reduceat(w.view(np.int64), p[:-1])],
                                          axis=1)) if r1 > r0 else torch.zeros((0, 2), torch.int64)
    full = shard.gather_rows(local, bounds)
    if rank == 0:
        fp, fi, fw = workloads.generate("cfg5", n=n, workers=2)
        if use_gpu:
            res = minhash_batch(fp, fi, fw, 128, HashFamily(4), bits=True, device="cuda:0")
            one = torch.cat([res.values, res.bits, res.status.to(torch.int64).unsqueeze(1)],
                            dim=1).cpu()
        else:
            one = torch.from_numpy(np.stack([np.diff(fp),
                                             np.add.reduceat(fw.view(np.int64), fp[:-1])], axis=1))
        q.put((rank, bool(torch.equal(full, one))))
    else:
        q.put((rank, True))
    dist.destroy_process_group()


def _run_ranks(world, use_gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_rows_worker, args=(r, world, port, q, use_gpu))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_rank_local_generation_gloo():
    """Per-rank generation over a lengths-only plan reproduces the one-process rows."""
    _run_ranks(2, use_gpu=False)


@pytest.mark.gpu
def test_rank_shards_byte_identical_to_one_launch_gloo():
    """Two ranks (gloo, sharing the one GPU; their kernels never wait on each
    other) sketch their own cfg5 row ranges; the gathered values, 1-bit words
    and statuses are byte-identical to a single launch over all rows."""
    _run_ranks(2, use_gpu=True)


def _lsh_rank_worker(rank, world, port, q):
    """The headline LSH workload's multi-GPU data path: cfg4 rows planned from
    the row lengths on t = L * K, each rank generating and keying only its own
    rows; the gathered keys equal one launch over the whole batch."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2005_11547_b200 import HashFamily, LshParams, lsh_batch
    n, prm = 3000, LshParams(100, 20)
    lens = workloads.lengths("cfg4", n)
    bounds = shard.plan_shards_lengths(lens, world, prm.L * prm.K)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    p, i, w = workloads.generate("cfg4", n=r1 - r0, start=r0, workers=2)
    res = lsh_batch(p, i, w, prm, HashFamily(3), device="cuda:0")
    local = torch.cat([res.keys, res.phi.to(torch.int64).unsqueeze(1),
                       res.status.to(torch.int64).unsqueeze(1)], dim=1).cpu()
    full = shard.gather_rows(local, bounds)
    ok = True
    if rank == 0:
        fp, fi, fw = workloads.generate("cfg4", n=n, workers=2)
        one = lsh_batch(fp, fi, fw, prm, HashFamily(3), device="cuda:0")
        ref = torch.cat([one.keys, one.phi.to(torch.int64).unsqueeze(1),
                         one.status.to(torch.int64).unsqueeze(1)], dim=1).cpu()
        ok = bool(torch.equal(full, ref))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_lsh_rank_shards_byte_identical_to_one_launch_gloo():
    """Two ranks (gloo, sharing the one GPU) key their own cfg4 row ranges; the
    gathered LSH keys, phi* and statuses are byte-identical to a single launch."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lsh_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_plan_shards_lsh_density():
    """LSH shards are balanced on t = L * K (the per-set term dominates for
    cfg4's fixed-size sets: equal row counts up to one row)."""
    lens = workloads.lengths("cfg4", 10001)
    b = shard.plan_shards_lengths(lens, 8, 2000)
    assert b[0] == 0 and b[-1] == 10001
    assert np.diff(b).max() - np.diff(b).min() <= 1
