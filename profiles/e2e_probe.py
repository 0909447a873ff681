"""Time dsk_minhash_csr_host on a workload through a given library (ctypes only).
usage: DSK_LIB_PATH=... python profiles/e2e_probe.py cfg5 2000000 [steps]"""
import ctypes, os, sys, time
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch
from paper_2005_11547_b200 import constants, workloads
name, n = sys.argv[1], int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = workloads.CONFIGS[name]
k = cfg.k[0]
indptr, ids, w = workloads.generate(name, n=n)
lib = ctypes.CDLL(os.environ["DSK_LIB_PATH"])
P = ctypes.c_void_p
tabs = constants.hash_tables(cfg.seed); cdf = constants.poisson1_cdf(); thr = constants.log2_thresholds()
ctx = P()
lib.dsk_ctx_create.argtypes = [ctypes.c_int, P, P, P, ctypes.POINTER(P)]
assert lib.dsk_ctx_create(0, tabs.ctypes.data, cdf.ctypes.data, thr.ctypes.data, ctypes.byref(ctx)) == 0
lib.dsk_minhash_csr_host.argtypes = [P, P, P, P, ctypes.c_int64, ctypes.c_int32, P, P, P, P, P]
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
for label, f in (("pinned", pin), ("pageable", lambda a: a)):
    hp, hi, hw = f(indptr), f(ids.view(np.int64)), f(w)
    ov, os_ = f(np.empty((n, k), np.int64)), f(np.empty(n, np.int32))
    def call():
        rc = lib.dsk_minhash_csr_host(ctx, hp.ctypes.data, hi.ctypes.data, hw.ctypes.data, n, k, ov.ctypes.data, None, os_.ctypes.data, None, None)
        assert rc == 0
    call()
    t0 = time.perf_counter()
    for _ in range(steps): call()
    dt = (time.perf_counter() - t0) / steps
    print(f"{os.path.basename(os.environ['DSK_LIB_PATH'])} {name} n={n} {label}: {dt*1e3:.1f} ms/step, bad={int((os_ != 0).sum())}", flush=True)
