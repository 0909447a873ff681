"""LSH on rows of skewed sizes (cfg5 rows): single-warp teams vs teams of 2 in the direct-only launch."""
import os, sys, time
import numpy as np, torch
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2005_11547_b200 import HashFamily, LshParams, lsh_batch, workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
indptr, ids, w = workloads.generate("cfg5", n=n)
dev = torch.device("cuda", 0)
p = torch.from_numpy(indptr).to(dev); i = torch.from_numpy(ids.view(np.int64)).to(dev); ww = torch.from_numpy(w).to(dev)
f = HashFamily(3)
for _ in range(2): r = lsh_batch(p, i, ww, LshParams(100, 20), f, check=False)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3): r = lsh_batch(p, i, ww, LshParams(100, 20), f, check=False)
torch.cuda.synchronize()
print(f"DSK_LSH_DG={os.environ.get('DSK_LSH_DG','default')} n={n} max nnz={int(np.diff(indptr).max())}: {(time.perf_counter()-t0)/3*1e3:.1f} ms/step, status!=0: {int((r.status!=0).sum())}")
