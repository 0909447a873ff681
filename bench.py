"""Benchmark: DartMinHash sketching throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2]
    python bench.py --impl reference ...      # CPU reference arm (oracle port)

A step = one pass of the hot path (dart_minhash for every set; lsh keys for
cfg4) over one batch of the workload, inputs resident in HBM.  Default
workload = BASELINE configs[1] (cfg2: 1e5 sets, nnz 1024, k 256), which fits
one GPU.  Under torchrun each rank sketches its own 1e5-set row block (weak
scaling, no data-path collective: the sets are independent).

Prints ONE JSON line (rank 0).  Extra keys:
  roofline      ALU bound: algorithmic hash evaluations (A + 2D + 2H per set,
                SURVEY.md §8(d)) per second vs the K0 peak hash rate measured
                in the same run; roofline_hbm gives the HBM view and
                roofline_issue the warp-instruction issue rate (the resource
                the kernel is actually bound by, ~65 % busy per ncu).
  cpu_baseline  the C oracle port of the reference on the host's cores.
  e2e           the same metric through the C ABI with host buffers
                (dsk_minhash_csr_host), H2D + D2H inside the timed region.
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
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--k", type=int, default=None, help="slot count (cfg3: 64/256/1024)")
    ap.add_argument("--sets", type=int, default=None, help="override sets per rank")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_rows(cfg, rank, n_per_rank):
    """CSR rows of this rank (optionally cached as .npy under $DSK_WL_CACHE)."""
    from paper_2005_11547_b200 import workloads
    cache = os.environ.get("DSK_WL_CACHE")
    if cache:
        base = os.path.join(cache, f"{cfg.name}_{rank * n_per_rank}_{n_per_rank}")
        if os.path.exists(base + "_w.npy"):
            return (np.load(base + "_p.npy"), np.load(base + "_i.npy"), np.load(base + "_w.npy"))
    out = workloads.generate(cfg.name, n=n_per_rank, start=rank * n_per_rank)
    if cache:
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


def cpu_model() -> str:
    """The host CPU's model string (BASELINE.md §2 asks for it next to the core count)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(cfg, k, indptr, ids, w, seconds, L=0, K=0):
    """The C oracle port of the reference on all host cores over a bounded sample."""
    from oracle.oracle import Oracle, default_threads
    orc = Oracle(cfg.seed)
    threads = default_threads()
    n = indptr.size - 1

    def run(rows):
        sub = (indptr[:rows + 1], ids[:indptr[rows]], w[:indptr[rows]])
        t0 = time.perf_counter()
        if cfg.kind == "lsh":
            orc.lsh_csr(*sub, L, K, nthreads=threads)
        else:
            orc.minhash_csr(*sub, k, nthreads=threads)
        return time.perf_counter() - t0

    probe = min(n, max(threads * 4, 64))
    dt = run(probe)
    rows = int(min(n, max(probe, probe * seconds / max(dt, 1e-6))))
    dt = run(rows)
    return {"value": rows / dt, "unit": "sketches/sec", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"first {rows} sets of the workload, {threads} threads, {dt:.1f} s"}


def reference_arm(args):
    """--impl reference: the oracle port (C restatement of the reference) on CPU."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2005_11547_b200 import workloads
    from oracle.oracle import Oracle, default_threads
    cfg = workloads.CONFIGS[args.workload]
    k = args.k or (cfg.k[0] if cfg.k else 0)
    threads = default_threads()
    orc = Oracle(cfg.seed)
    # bounded sample per step: ~args.cpu_seconds/steps of CPU work
    n_avail = min(cfg.n, 20000)
    indptr, ids, w = workloads.generate(cfg.name, n=n_avail)

    def step(rows):
        sub = (indptr[:rows + 1], ids[:indptr[rows]], w[:indptr[rows]])
        if cfg.kind == "lsh":
            orc.lsh_csr(*sub, cfg.L, cfg.K, nthreads=threads)
        else:
            orc.minhash_csr(*sub, k, nthreads=threads)

    probe = min(n_avail, threads * 8)
    t0 = time.perf_counter()
    step(probe)
    dt = time.perf_counter() - t0
    per_step = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    rows = int(min(n_avail, max(probe, probe * per_step / max(dt, 1e-6))))
    for _ in range(args.warmup):
        step(min(rows, probe))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step(rows)
        times.append(time.perf_counter() - t0)
    ms = 1000.0 * sum(times) / len(times)
    value = rows / (ms / 1000.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sketches/sec",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64/f64",
        "data": "synthetic",
        "config": {"workload": cfg.name, "description": cfg.description, "k": k,
                   "sets_per_step": rows},
        "cpu_baseline": {"value": value, "unit": "sketches/sec", "cores": threads,
                         "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"first {rows} sets of {cfg.name} per step, {threads} threads "
                                   "(C restatement of the reference, oracle/)"},
        "e2e": {"value": value, "unit": "sketches/sec", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2005_11547_b200 import HashFamily, LshParams, _lib, lsh_batch, minhash_batch
    from paper_2005_11547_b200 import workloads

    rank, world, local = dist_env()
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
    cfg = workloads.CONFIGS[args.workload]
    k = args.k or (cfg.k[0] if cfg.k else 0)
    n = args.sets or cfg.n
    indptr, ids, w = workload_rows(cfg, rank, n)
    fam = HashFamily(cfg.seed)
    lib = _lib.load()
    p_d = torch.from_numpy(indptr).to(dev)
    i_d = torch.from_numpy(ids.view(np.int64)).to(dev)
    w_d = torch.from_numpy(w).to(dev)
    nnz = int(indptr[-1])
    onebit = cfg.onebit

    def step():
        if cfg.kind == "lsh":
            return lsh_batch(p_d, i_d, w_d, LshParams(cfg.L, cfg.K), fam, check=False)
        return minhash_batch(p_d, i_d, w_d, k, fam, bits=onebit, check=False)

    for _ in range(max(args.warmup, 3)):
        res = step()
    torch.cuda.synchronize()
    status = res.status.cpu().numpy()
    stats = res.stats.cpu().numpy().view(np.uint32).astype(np.int64)
    bad = int((status != 0).sum())

    # K0: peak hash rates on this device (roofline denominators)
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    ctx = fam.context(dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)

    def hash_rate(mode, iters):
        done = ctypes.c_int64()
        lib.dsk_hash_peak(ctx, mode, 16, ctypes.c_void_p(sink.data_ptr()), ctypes.byref(done),
                          stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.dsk_hash_peak(ctx, mode, iters, ctypes.c_void_p(sink.data_ptr()), ctypes.byref(done),
                          stream)
        e1.record()
        torch.cuda.synchronize()
        return done.value / (e0.elapsed_time(e1) / 1000.0)

    peak_hps = hash_rate(0, 256)          # full 22-lookup tabulation hash (reference's unit)
    peak_hoisted_hps = hash_rate(1, 4096)  # one lookup + finalizer (hoisted lower bound on cost)

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
    ms = start.elapsed_time(end) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    # work units: areas A, candidate darts D, hits H at phi*
    A, D, H = stats[:, 0].sum(), stats[:, 1].sum(), stats[:, 2].sum()
    hashes = A + 2 * D + 2 * H + (cfg.L * cfg.K * n if cfg.kind == "lsh" else 0)
    tot = torch.tensor([float(n), float(H), float(hashes)], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(tot)
    sets_all, hits_all, hashes_all = (float(x) for x in tot.tolist())
    sec = ms_max / 1000.0
    value = sets_all / sec
    out_bytes = n * (8 * k + 8 * ((k + 63) // 64) * onebit + 4 + 4 + 16) if cfg.kind != "lsh" \
        else n * (8 * cfg.L + 24)
    hbm_bytes = 16 * nnz + 8 * (n + 1) + out_bytes
    peak_hbm = 6543.1
    try:
        peak_hbm = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass

    # e2e through the C ABI with host (pinned) buffers
    e2e = None
    if not args.no_e2e:
        pin_p = torch.from_numpy(indptr).pin_memory()
        pin_i = torch.from_numpy(ids.view(np.int64)).pin_memory()
        pin_w = torch.from_numpy(w).pin_memory()
        lsh = cfg.kind == "lsh"
        o_v = torch.empty((n, cfg.L if lsh else k), dtype=torch.int64).pin_memory()
        o_s = torch.empty(n, dtype=torch.int32).pin_memory()
        words = (k + 63) // 64
        o_b = torch.empty((n, words), dtype=torch.int64).pin_memory() if onebit else None
        api = "dsk_lsh_csr_host" if lsh else "dsk_minhash_csr_host"
        P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731

        def host_call():
            if lsh:
                rc = lib.dsk_lsh_csr_host(ctx, P(pin_p), P(pin_i), P(pin_w), n, cfg.L, cfg.K, 0,
                                          P(o_v), None, P(o_s), None, None)
            else:
                rc = lib.dsk_minhash_csr_host(ctx, P(pin_p), P(pin_i), P(pin_w), n, k, P(o_v),
                                              P(o_b), P(o_s), None, None)
            _lib.check(rc, api)

        host_call()
        if world > 1:
            dist.barrier()
        b0 = lib.dsk_h2d_bytes()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            host_call()
        dt = (time.perf_counter() - t0) / args.steps
        h2d_copied = (lib.dsk_h2d_bytes() - b0) // args.steps
        tt = torch.tensor([dt], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        h2d = int(h2d_copied)  # as counted by the library (dsk_h2d_bytes)
        d2h = o_v.numel() * 8 + o_s.numel() * 4 + (o_b.numel() * 8 if o_b is not None else 0)
        e2e = {"value": sets_all / dt, "unit": "sketches/sec", "ms_per_step": dt * 1000.0,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "api": f"{api} (C ABI, pinned host buffers)",
               "input_bytes_per_step": int(indptr.nbytes + ids.nbytes + w.nbytes)}
        assert (o_s.numpy() == 0).all()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, k, indptr, ids, w, args.cpu_seconds, cfg.L, cfg.K)

    if rank == 0:
        traffic = None
        issue = None
        tkey = cfg.name if args.k is None else f"{cfg.name}_k{k}"
        tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
        entry = json.load(open(tpath)).get(tkey) if os.path.exists(tpath) else None
        if entry and args.sets is None and "bytes_per_launch" in entry:
            traffic = {"bytes_per_launch": entry["bytes_per_launch"],
                       "algorithmic_bytes_per_launch": hbm_bytes,
                       "source": entry["source"]}
        if entry and "warp_instructions_per_set" in entry and clk.get("sm_mhz"):
            # the binding resource: warp-instruction issue (4 per SM per clock)
            ips = entry["warp_instructions_per_set"] * n / (ms_max / 1e3)
            peak_ips = 4.0 * torch.cuda.get_device_properties(dev).multi_processor_count * \
                float(clk["sm_mhz"]) * 1e6
            issue = {"bound": "issue", "achieved": ips / 1e9, "peak": peak_ips / 1e9,
                     "unit": "G warp-inst/s", "frac": ips / peak_ips,
                     "note": "ncu instruction count per set (profiles/ncu_traffic.json) x sets / "
                             "kernel time, against 4 issues/clk/SM at the sampled SM clock"}
        achieved = hashes_all / sec / 1e9
        peak = peak_hps / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": "sketches/sec", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64/f64", "data": "synthetic",
            "config": {"workload": cfg.name, "description": cfg.description,
                       "sets_per_gpu": n, "nnz_per_gpu": nnz, "k": k,
                       "L": cfg.L or None, "K": cfg.K or None, "onebit": onebit,
                       "l2": f"inputs larger than L2 ({hbm_bytes / 1e9:.2f} GB per GPU per step)",
                       "parallelism": f"row shards x{world}, no collective"},
            "darts_per_sec": hits_all / sec,
            "hash_evals_per_sec": hashes_all / sec,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak,
                         "unit": "Ghash/s", "frac": achieved / peak, "traffic": traffic,
                         "peak_hoisted": peak_hoisted_hps / 1e9,
                         "frac_hoisted": achieved / (peak_hoisted_hps / 1e9),
                         "note": "achieved = algorithmic hash evaluations A+2D+2H per set "
                                 "(SURVEY 8d; each one 22-byte tabulation hash + splitmix64, "
                                 "ref/randomness.py:121-131) per second of the sketch kernel; "
                                 "peak = K0 mode 0, that full 22-lookup hash on all SMs, "
                                 "measured this run; peak_hoisted = K0 mode 1 (1 lookup + "
                                 "finalizer), the rate if every hash were fully hoisted"},
            "roofline_hbm": {"bound": "hbm", "achieved": hbm_bytes / sec / 1e9 * 1.0,
                             "peak": peak_hbm, "unit": "GB/s",
                             "frac": hbm_bytes / sec / 1e9 / peak_hbm,
                             "note": "16 B/nonzero + 8 B/set + outputs; peak = MEASURED_PEAKS.json"},
            "roofline_issue": issue,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk,
            "status_nonzero": bad,
            "phi_hist": np.bincount(stats[:, 3]).tolist(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
