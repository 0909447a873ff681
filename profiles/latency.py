"""Small-batch latency: single-set API calls (dart_minhash / lsh_key, wall
clock incl. copies) and device-resident batches of 1 / 100 / 1000 sets
(CUDA events).  Run with DSK_NO_WAVE=1 to compare against the large-batch
team shape."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_11547_b200 import (HashFamily, LshParams, WeightedSet, dart_minhash,  # noqa: E402
                                   lsh_batch, lsh_key, minhash_batch, workloads)

dev = torch.device("cuda", 0)
out = {"no_wave": bool(os.environ.get("DSK_NO_WAVE"))}
h = HashFamily(1)
p, i, w = workloads.generate("cfg2", n=1000)
x = WeightedSet.from_arrays(i[:p[1]], w[:p[1]])
for _ in range(3):
    dart_minhash(x, 256, h)
t = time.perf_counter()
for _ in range(20):
    dart_minhash(x, 256, h)
out["dart_minhash_cfg2_ms"] = (time.perf_counter() - t) / 20 * 1e3
p4, i4, w4 = workloads.generate("cfg4", n=10)
x4 = WeightedSet.from_arrays(i4[:p4[1]], w4[:p4[1]])
h4 = HashFamily(3)
for _ in range(3):
    lsh_key(x4, LshParams(100, 20), h4)
t = time.perf_counter()
for _ in range(20):
    lsh_key(x4, LshParams(100, 20), h4)
out["lsh_key_cfg4_ms"] = (time.perf_counter() - t) / 20 * 1e3


def dev_batch(cfg, n, k=None, lsh=None):
    pp, ii, ww = workloads.generate(cfg, n=n)
    pd = torch.from_numpy(pp).to(dev)
    idd = torch.from_numpy(ii.view(np.int64)).to(dev)
    wd = torch.from_numpy(ww).to(dev)
    fam = HashFamily(workloads.CONFIGS[cfg].seed)

    def call():
        if lsh:
            return lsh_batch(pd, idd, wd, lsh, fam, check=False)
        return minhash_batch(pd, idd, wd, k, fam, check=False)
    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        call()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10


for n in (1, 100, 1000):
    out[f"cfg2_batch{n}_ms"] = dev_batch("cfg2", n, k=256)
out["cfg1_batch1000_ms"] = dev_batch("cfg1", 1000, k=64)
out["cfg4_batch100_ms"] = dev_batch("cfg4", 100, lsh=LshParams(100, 20))
print(json.dumps(out))
