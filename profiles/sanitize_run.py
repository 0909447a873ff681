"""Small end-to-end run of every kernel for compute-sanitizer (one tool per call)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_11547_b200 import (HashFamily, LshParams, bottom_k_batch, darts_batch,  # noqa
                                   lsh_batch, minhash_batch, workloads)

p, i, w = workloads.generate("cfg1", n=40)
f = HashFamily(0)
minhash_batch(p, i, w, 64, f, bits=True)
minhash_batch(p, i, w, 1024, f)          # multi-warp teams
p3, i3, w3 = workloads.generate("cfg2", n=8)
minhash_batch(p3, i3, w3, 256, f)        # rank depth 1: region path
lsh_batch(p, i, w, LshParams(100, 20), f, fps=True)
bottom_k_batch(p, i, w, 17, f)
darts_batch(p, i, w, 331, np.full(40, 1.0 / 128), f)
print("sanitize run ok")
