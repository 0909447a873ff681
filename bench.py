"""Benchmark: DartMinHash sketching throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4]
    python bench.py --impl reference ...      # CPU reference arm

A step = one pass of the hot path over one batch of the workload with the
inputs resident in HBM: `lsh_batch` (ref/annindex.py:64-82 + mix64 per table)
for cfg4, `minhash_batch` (ref/sketching.py:115-123, + the 1-bit epilogue for
cfg3) otherwise.  The default workload is cfg4 (BASELINE configs[3]: 1e6 sets,
nnz 128, LogNormal(0,1), (L,K) = (100,20)), the largest configuration whose
sets fit one GPU per the round-1 verdict; cfg1-cfg5 are all selectable, cfg5
at its full 1e7 sets.

Under torchrun (one rank per GPU) the batch is the SAME n sets for every N
(strong scaling): the row ranges come from `shard.plan_shards_lengths` over
the workload's row lengths (computed without generating the rows), each rank
generates and sketches only its own range, and there is no data-path
collective (the sets are independent).  The timed region is
bracketed by barrier + synchronize; the time is the max over ranks.

Prints ONE JSON line (rank 0).  Extra keys:
  roofline          the binding resource, warp-instruction issue: ncu's
                    instruction count per set for this workload
                    (profiles/ncu_traffic.json, same command captured under
                    ncu) x sets / kernel time, against 4 issues/clk/SM at the
                    SM clock sampled during the timed region; `traffic` = the
                    same capture's DRAM bytes scaled to this launch.
  roofline_useful   the useful-work lower bound: the areas, candidate darts,
                    hits (and mix64 steps) of this step, each priced at the
                    rate the K0 unit microbenchmarks reach on this GPU in this
                    run with no enumeration bookkeeping; frac = that time /
                    the kernel time.
  roofline_hbm      CSR bytes + outputs over the measured copy bandwidth.
  cpu_baseline      the unmodified Python reference (baseline/_ref) on every
                    host core (multiprocessing) over a bounded
                    sample; `cpu_port` = the C restatement (oracle/) likewise.
  e2e               the same metric through the C ABI with host buffers
                    (dsk_lsh_csr_host / dsk_minhash_csr_host), H2D + D2H in the
                    timed region, pinned buffers; `e2e_pageable` = the same call
                    with plain numpy arrays (the INTEGRATION.md binding).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "sketches/sec"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--k", type=int, default=None, help="slot count (cfg3: 64/256/1024)")
    ap.add_argument("--sets", type=int, default=None, help="override the workload's set count")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    return rank, world, local, local_world


def host_cores() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def density(cfg, k):
    from paper_2005_11547_b200.constants import minhash_density
    return cfg.L * cfg.K if cfg.kind == "lsh" else minhash_density(k)


def shard_bounds(cfg, n_total, world, k):
    """Row ranges of the ranks: balanced by the per-row cost model over the
    workload's row lengths (drawn without generating the rows)."""
    from paper_2005_11547_b200 import shard, workloads
    lens = workloads.lengths(cfg.name, n_total)
    return shard.plan_shards_lengths(lens, world, density(cfg, k))


def rows_of(cfg, r0, r1, workers):
    """CSR rows [r0, r1) of the workload (optionally cached under $DSK_WL_CACHE)."""
    from paper_2005_11547_b200 import workloads
    cache = os.environ.get("DSK_WL_CACHE")
    base = os.path.join(cache, f"{cfg.name}_{r0}_{r1 - r0}") if cache else None
    if base and os.path.exists(base + "_w.npy"):
        return (np.load(base + "_p.npy"), np.load(base + "_i.npy"), np.load(base + "_w.npy"))
    out = workloads.generate(cfg.name, n=r1 - r0, start=r0, workers=workers)
    if base:
        os.makedirs(cache, exist_ok=True)
        for suffix, arr in zip(("_p", "_i", "_w"), out):
            np.save(base + suffix + ".npy", arr)
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------ CPU baselines

def cpu_port(cfg, k, indptr, ids, w, seconds):
    """The C restatement of the reference (oracle/, test infrastructure) on
    all host threads over a bounded sample of the same rows."""
    from oracle.oracle import Oracle, default_threads
    from baseline.pyref import cpu_model
    orc = Oracle(cfg.seed)
    threads = default_threads()
    n = indptr.size - 1

    def run(rows):
        sub = (indptr[:rows + 1], ids[:indptr[rows]], w[:indptr[rows]])
        t0 = time.perf_counter()
        if cfg.kind == "lsh":
            orc.lsh_csr(*sub, cfg.L, cfg.K, nthreads=threads)
        else:
            orc.minhash_csr(*sub, k, nthreads=threads)
        return time.perf_counter() - t0

    probe = min(n, max(threads * 4, 64))
    dt = run(probe)
    rows = int(min(n, max(probe, probe * seconds / max(dt, 1e-6))))
    dt = run(rows)
    return {"value": rows / dt, "unit": "sketches/sec", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"first {rows} sets of {cfg.name} (this rank's rows), {threads} threads, "
                      f"{dt:.1f} s"}


def cpu_reference(cfg, k, indptr, ids, w, seconds, pool=None):
    """The unmodified Python reference on every host core (baseline/pyref.py)."""
    from baseline import pyref
    if not pyref.available():
        return None
    own = pool is None
    pool = pool or pyref.PyRefPool()
    try:
        rate, rows, _ = pool.timed_sample(cfg.kind, cfg.seed, k, cfg.L, cfg.K, cfg.onebit,
                                          indptr, ids, w, seconds)
    finally:
        if own:
            pool.close()
    call = ("lsh_key + mix64 per table" if cfg.kind == "lsh" else
            "dart_minhash" + (" + one_bit" if cfg.onebit else ""))
    return {"value": rate, "unit": "sketches/sec", "cores": pool.workers, "kind": "reference",
            "cpu_model": pyref.cpu_model(),
            "sample": f"first {rows} sets of {cfg.name}, unmodified dartsketch 0.1.0 "
                      f"({call}), {pool.workers} processes, ~{seconds:.0f} s busy each"}


def reference_arm(args):
    """--impl reference: the reference's own CPU implementation of the path on
    the host's cores -- the unmodified Python package (baseline/_ref) when it
    is installed, else the C restatement (oracle/) -- over a bounded sample of
    the workload per step.  Rank 0 only."""
    rank, world, _, _ = dist_env()
    if rank != 0:
        return
    from baseline import pyref
    from paper_2005_11547_b200 import workloads
    cfg = workloads.CONFIGS[args.workload]
    k = args.k or (cfg.k[0] if cfg.k else 0)
    n_avail = min(args.sets or cfg.n, 20000)
    indptr, ids, w = workloads.generate(cfg.name, n=n_avail)
    per_step = max(2.0, 90.0 / max(1, args.steps + args.warmup))
    port = cpu_port(cfg, k, indptr, ids, w, min(per_step, 5.0))
    if pyref.available():
        pool = pyref.PyRefPool()
        probe = min(n_avail, 2 * pool.workers)
        rate, _ = pool.run(cfg.kind, cfg.seed, k, cfg.L, cfg.K, cfg.onebit, indptr, ids, w, probe)
        rows = int(min(n_avail, max(probe, rate * per_step)))
        run = lambda m: pool.run(cfg.kind, cfg.seed, k, cfg.L, cfg.K, cfg.onebit,  # noqa: E731
                                 indptr, ids, w, m)[0]
        kind, cores = "reference", pool.workers
        sample = (f"first {rows} sets of {cfg.name} per step, unmodified dartsketch 0.1.0 "
                  f"(baseline/_ref), {cores} processes")
    else:
        from oracle.oracle import Oracle, default_threads
        orc = Oracle(cfg.seed)
        cores = default_threads()
        pool = None

        def run(m):
            sub = (indptr[:m + 1], ids[:indptr[m]], w[:indptr[m]])
            t0 = time.perf_counter()
            if cfg.kind == "lsh":
                orc.lsh_csr(*sub, cfg.L, cfg.K, nthreads=cores)
            else:
                orc.minhash_csr(*sub, k, nthreads=cores)
            return m / (time.perf_counter() - t0)
        rows = int(min(n_avail, port["value"] * per_step))
        kind = "port"
        sample = f"first {rows} sets of {cfg.name} per step, {cores} threads (C restatement, oracle/)"
    for _ in range(args.warmup):
        run(min(rows, 2 * cores))
    rates = [run(rows) for _ in range(args.steps)]
    if pool is not None:
        pool.close()
    ms = 1000.0 * statistics.mean(rows / r for r in rates)
    value = rows / (ms / 1000.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sketches/sec",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64/f64", "data": "synthetic",
        "config": {"workload": cfg.name, "description": cfg.description, "k": k,
                   "L": cfg.L or None, "K": cfg.K or None, "sets_per_step": rows},
        "cpu_baseline": {"value": value, "unit": "sketches/sec", "cores": cores, "kind": kind,
                         "cpu_model": pyref.cpu_model(), "sample": sample},
        "cpu_port": port,
        "e2e": {"value": value, "unit": "sketches/sec", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm

def unit_rates(lib, ctx, dev, stream):
    """K0 microbenchmarks (units/s on this GPU): 0 reference hash, 1 hoisted
    hash, 2 area, 3 candidate dart, 4 hit, 5 mix64 step."""
    import torch
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    iters = {0: 256, 1: 4096, 2: 2048, 3: 2048, 4: 1024, 5: 1024}
    rates = {}
    for mode, it in iters.items():
        done = ctypes.c_int64()
        lib.dsk_hash_peak(ctx, mode, 16, ctypes.c_void_p(sink.data_ptr()), ctypes.byref(done),
                          stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.dsk_hash_peak(ctx, mode, it, ctypes.c_void_p(sink.data_ptr()), ctypes.byref(done),
                          stream)
        e1.record()
        torch.cuda.synchronize()
        rates[mode] = done.value / (e0.elapsed_time(e1) / 1000.0)
    return rates


def ncu_entry(cfg, k, explicit_k):
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    key = cfg.name if not explicit_k else f"{cfg.name}_k{k}"
    return json.load(open(path)).get(key)


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    from paper_2005_11547_b200 import workloads
    rank, world, local, local_world = dist_env()
    cfg = workloads.CONFIGS[args.workload]
    k = args.k or (cfg.k[0] if cfg.k else 0)
    n_total = args.sets or cfg.n
    # shard plan + this rank's rows, before CUDA is touched (the generator
    # forks host workers); the ranks of a node share its cores
    bounds = shard_bounds(cfg, n_total, world, k)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    t_gen = time.perf_counter()
    indptr, ids, w = rows_of(cfg, r0, r1, max(1, host_cores() // max(1, local_world)))
    t_gen = time.perf_counter() - t_gen

    import torch
    import torch.distributed as dist

    from paper_2005_11547_b200 import HashFamily, LshParams, _lib, lsh_batch, minhash_batch

    # one rank per GPU; DSK_DIST_BACKEND=gloo (+ more ranks than GPUs) is only
    # for exercising the multi-rank code path on a one-GPU box, never timed
    backend = os.environ.get("DSK_DIST_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    red_dev = dev if backend == "nccl" else torch.device("cpu")  # reduction tensors
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def all_max(x):
        t = torch.tensor([float(x)], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def all_sum(xs):
        t = torch.tensor([float(x) for x in xs], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t)
        return [float(x) for x in t.tolist()]

    n = r1 - r0
    nnz = int(indptr[-1])
    fam = HashFamily(cfg.seed)
    lib = _lib.load()
    p_d = torch.from_numpy(indptr).to(dev)
    i_d = torch.from_numpy(ids.view(np.int64)).to(dev)
    w_d = torch.from_numpy(w).to(dev)
    onebit = cfg.onebit
    lsh = cfg.kind == "lsh"

    def step():
        if lsh:
            return lsh_batch(p_d, i_d, w_d, LshParams(cfg.L, cfg.K), fam, check=False)
        return minhash_batch(p_d, i_d, w_d, k, fam, bits=onebit, check=False)

    for _ in range(max(args.warmup, 3)):
        res = step()
    torch.cuda.synchronize()
    status = res.status.cpu().numpy()
    stats = res.stats.cpu().numpy().view(np.uint32).astype(np.int64)
    bad = int((status != 0).sum())

    ctx = fam.context(dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    rates = unit_rates(lib, ctx, dev, stream)

    clocks = ClockSampler(local_dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.dsk_launch_count()
    start.record()
    for _ in range(args.steps):
        res = step()
    end.record()
    launches = int(lib.dsk_launch_count() - launches0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_local = start.elapsed_time(end) / args.steps
    ms_max = all_max(ms_local)
    sec = ms_max / 1000.0

    # work units: areas A, candidate darts D, hits H at phi*
    A, D, H = (float(stats[:, c].sum()) for c in range(3))
    LK = float(cfg.L * cfg.K * n) if lsh else 0.0
    hashes = A + 2 * D + 2 * H + LK
    sets_all, A_all, D_all, H_all, LK_all, hashes_all, bad_all = all_sum(
        [n, A, D, H, LK, hashes, bad])
    value = sets_all / sec
    words = (k + 63) // 64
    out_bytes = n * (8 * cfg.L + 24) if lsh else \
        n * (8 * k + 8 * words * onebit + 4 + 4 + 16)
    hbm_bytes = 16 * nnz + 8 * (n + 1) + out_bytes
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    peak_hbm = float(peaks.get("hbm_gbs", 6543.1))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    # ------------------------------------------------------------ e2e legs
    e2e = e2e_pageable = None
    if not args.no_e2e:
        api = "dsk_lsh_csr_host" if lsh else "dsk_minhash_csr_host"
        P = lambda a: ctypes.c_void_p(a.ctypes.data) if a is not None else None  # noqa: E731

        def host_call(hp, hi, hw, ov, ob, os_):
            if lsh:
                rc = lib.dsk_lsh_csr_host(ctx, P(hp), P(hi), P(hw), n, cfg.L, cfg.K, 0,
                                          P(ov), None, P(os_), None, None)
            else:
                rc = lib.dsk_minhash_csr_host(ctx, P(hp), P(hi), P(hw), n, k, P(ov), P(ob),
                                              P(os_), None, None)
            _lib.check(rc, api)

        def timed(bufs, label):
            host_call(*bufs)
            if world > 1:
                dist.barrier()
            b0 = lib.dsk_h2d_bytes()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                host_call(*bufs)
            dt = all_max((time.perf_counter() - t0) / args.steps)
            h2d = (lib.dsk_h2d_bytes() - b0) // args.steps
            ov, ob, os_ = bufs[3:]
            d2h = ov.nbytes + os_.nbytes + (ob.nbytes if ob is not None else 0)
            assert (os_ == 0).all(), "status != 0 on the host-buffer path"
            return {"value": sets_all / dt, "unit": "sketches/sec", "ms_per_step": dt * 1000.0,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "api": f"{api} (C ABI, {label})"}

        cols = cfg.L if lsh else k
        in_bytes = indptr.nbytes + ids.nbytes + w.nbytes
        out_b = n * cols * 8 + n * 4 + (n * words * 8 if onebit else 0)
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except ImportError:
            avail = 1 << 40
        if (in_bytes + out_b) * local_world < 0.3 * avail:
            pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
            bufs = (pin(indptr), pin(ids.view(np.int64)), pin(w),
                    pin(np.empty((n, cols), np.int64)),
                    pin(np.empty((n, words), np.int64)) if onebit else None,
                    pin(np.empty(n, np.int32)))
            e2e = timed(bufs, "pinned host buffers")
            del bufs
        pbufs = (indptr, ids, w, np.empty((n, cols), np.uint64),
                 np.empty((n, words), np.uint64) if onebit else None, np.empty(n, np.int32))
        e2e_pageable = timed(pbufs, "plain numpy arrays, the INTEGRATION.md binding")
        if e2e is None:
            e2e = e2e_pageable

    cpu = port = None
    if rank == 0 and world == 1 and not args.no_cpu:
        port = cpu_port(cfg, k, indptr, ids, w, args.cpu_seconds)
        cpu = cpu_reference(cfg, k, indptr, ids, w, args.cpu_seconds) or port

    if rank == 0:
        entry = ncu_entry(cfg, k, args.k is not None)
        issue = traffic = None
        if entry and entry.get("dram_bytes_per_set"):
            traffic = entry["dram_bytes_per_set"] * n
        if entry and clk.get("sm_mhz"):
            ips = entry["warp_instructions_per_set"] * n / sec
            peak_ips = 4.0 * sms * float(clk["sm_mhz"]) * 1e6
            issue = {"bound": "issue", "achieved": ips / 1e9, "peak": peak_ips / 1e9,
                     "unit": "G warp-inst/s", "frac": ips / peak_ips, "traffic": traffic,
                     "algorithmic_bytes": hbm_bytes,
                     "source": entry.get("source"),
                     "note": "the binding resource (SURVEY 8(d), north_star: INT/hash-ALU "
                             "issue rate): ncu smsp__inst_executed per set of this workload's "
                             "kernel x sets / kernel time, against 4 warp-instructions/clk/SM x "
                             f"{sms} SMs at the sampled SM clock; traffic = that capture's "
                             "dram__bytes_read+write per set x sets (bytes per launch)"}
        useful_s = (A_all / rates[2] + D_all / rates[3] + H_all / rates[4] +
                    (LK_all / rates[5] if lsh else 0.0)) / world
        useful = {"bound": "alu-useful", "achieved": useful_s * 1000.0, "peak": ms_max,
                  "unit": "ms/step", "frac": useful_s / sec,
                  "unit_rates_G_per_s": {"ref_hash": rates[0] / 1e9, "hoisted_hash": rates[1] / 1e9,
                                         "area": rates[2] / 1e9, "dart": rates[3] / 1e9,
                                         "hit": rates[4] / 1e9, "mix64_step": rates[5] / 1e9},
                  "note": "lower bound on the step time: A areas / area rate + D darts / dart "
                          "rate + H hits / hit rate (+ L*K mix64 steps), each rate from the K0 "
                          "unit microbenchmark (all SMs, no enumeration bookkeeping) in this "
                          "run; frac = bound / measured kernel time"}
        line = {
            "metric": METRIC, "value": value, "unit": "sketches/sec", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u64/f64", "data": "synthetic",
            "config": {"workload": cfg.name, "description": cfg.description,
                       "sets": int(n_total), "sets_rank0": n, "nnz_rank0": nnz, "k": k or None,
                       "L": cfg.L or None, "K": cfg.K or None, "onebit": onebit,
                       "l2": f"inputs larger than L2 ({hbm_bytes / 1e9:.2f} GB per GPU per step)",
                       "parallelism": f"row shards x{world} (plan_shards_lengths), no collective",
                       "host_generation_s": round(t_gen, 2)},
            "darts_per_sec": H_all / sec,
            "hash_evals_per_sec": hashes_all / sec,
            "roofline": issue,
            "roofline_useful": useful,
            "roofline_hbm": {"bound": "hbm", "achieved": hbm_bytes / sec / 1e9, "peak": peak_hbm,
                             "unit": "GB/s", "frac": hbm_bytes / sec / 1e9 / peak_hbm,
                             "note": "16 B/nonzero + 8 B/set + outputs (rank 0); peak = "
                                     "MEASURED_PEAKS.json hbm_gbs"},
            "ref_hash_rate_G_per_s": rates[0] / 1e9,
            "e2e": e2e,
            "e2e_pageable": e2e_pageable,
            "cpu_baseline": cpu,
            "cpu_port": port,
            "gpu_launches": launches,
            "clocks": clk,
            "status_nonzero": int(bad_all),
            "phi_hist": np.bincount(stats[:, 3]).tolist(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
