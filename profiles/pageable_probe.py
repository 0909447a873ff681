"""e2e of dsk_minhash_csr_host with pageable numpy inputs vs pinned ones (cfg2)."""
import ctypes, json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_11547_b200 import HashFamily, _lib, workloads

indptr, ids, w = workloads.generate("cfg2", n=100000)
fam = HashFamily(1)
lib = _lib.load()
ctx = fam.context(torch.device("cuda", 0))
P = ctypes.c_void_p
n, k = indptr.size - 1, 256
res = {}
for name in ("pageable", "pinned", "pinned_in_pageable_out"):
    if name == "pinned_in_pageable_out":
        ip = torch.from_numpy(indptr).pin_memory().numpy()
        ii = torch.from_numpy(ids.view(np.int64)).pin_memory().numpy().view(np.uint64)
        ww = torch.from_numpy(w).pin_memory().numpy()
        vals = np.empty((n, k), dtype=np.int64)
        st = np.empty(n, dtype=np.int32)
    elif name == "pinned":
        ip = torch.from_numpy(indptr).pin_memory().numpy()
        ii = torch.from_numpy(ids.view(np.int64)).pin_memory().numpy().view(np.uint64)
        ww = torch.from_numpy(w).pin_memory().numpy()
        vals = torch.empty((n, k), dtype=torch.int64).pin_memory().numpy()
        st = torch.empty(n, dtype=torch.int32).pin_memory().numpy()
    else:
        ip, ii, ww = indptr, ids, w
        vals = np.empty((n, k), dtype=np.int64)
        st = np.empty(n, dtype=np.int32)
    def call():
        rc = lib.dsk_minhash_csr_host(ctx, P(ip.ctypes.data), P(ii.ctypes.data), P(ww.ctypes.data),
                                      n, k, P(vals.ctypes.data), None, P(st.ctypes.data), None, None)
        assert rc == 0
    call()
    t = time.perf_counter()
    for _ in range(3):
        call()
    res[name] = (time.perf_counter() - t) / 3 * 1e3
print(json.dumps(res))
