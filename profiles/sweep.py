"""Build tuning variants of libdsk_b200.so (in-tree, travel with gpurun) and
time each on the quick workload list.  Variants are compile-time defines of
csrc/dsk_engine.cuh / dsk_kernels.cu / dsk_lsh_kernel.cuh (DSK_DIRECT,
DSK_RUN, DSK_REFILL, DSK_FUSE, DSK_OPAQUE, DSK_LPT, DSK_LSH_CLOSE, ...).

  python profiles/sweep.py build            # here (nvcc, no GPU)
  python profiles/sweep.py run [workloads]  # on the GPU box
"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
VDIR = os.path.join(REPO, "paper_2005_11547_b200", "variants")

VARIANTS = {
    # compile-time variants measured this round (DESIGN.md §9 lists the
    # outcomes); the defaults of csrc/dsk_engine.cuh / dsk_kernels.cu won
    "default": {},
    "direct2": {"DSK_DIRECT": 2},
    "run4": {"DSK_RUN": 4},
    "refill12": {"DSK_REFILL": 12},
    "no_opaque": {"DSK_OPAQUE": 0},
    "no_lpt": {"DSK_LPT": 0},
    "lsh_nofuse": {"DSK_LSH_FUSE": 0},
    "pt_smem": {"DSK_PT_IMM": 0},
}
WORKLOADS = ["cfg2", "cfg3 --k 64", "cfg3 --k 256", "cfg3 --k 1024", "cfg4",
             "cfg5 --sets 1000000"]


def build():
    from paper_2005_11547_b200 import _lib
    os.makedirs(VDIR, exist_ok=True)
    for name, d in VARIANTS.items():
        out = os.path.join(VDIR, f"libdsk_{name}.so")
        _lib.build(out=out, defines=d)
        print("built", out, flush=True)


def run(names, workloads):
    res = {}
    for name in names:
        lib = os.path.join(VDIR, f"libdsk_{name}.so")
        env = dict(os.environ, DSK_LIB_PATH=lib, DSK_WL_CACHE="/tmp/dsk_wl")
        for wl in workloads:
            cmd = [sys.executable, os.path.join(REPO, "bench.py"), "--steps", "3", "--warmup", "3",
                   "--no-cpu", "--no-e2e", "--workload"] + wl.split()
            p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
            try:
                d = json.loads(p.stdout.strip().splitlines()[-1])
                res[(name, wl)] = d["ms_per_step"]
                ok = d["status_nonzero"] == 0
            except Exception:
                res[(name, wl)] = None
                ok = False
            print(f"{name:10s} {wl:22s} {res[(name, wl)]}  ok={ok}", flush=True)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        wls = sys.argv[2:] or WORKLOADS
        run(list(VARIANTS), wls)
