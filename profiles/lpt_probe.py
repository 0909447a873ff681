import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2005_11547_b200 import HashFamily, minhash_batch, workloads
p, i, w = workloads.generate("cfg5", n=1000000)
nnz = np.diff(p)
order = np.argsort(-nnz, kind="stable")
sp, si, sw = workloads.subset(p, i, w, order)
dev = torch.device("cuda", 0)
fam = HashFamily(4)
def run(pp, ii, ww):
    P = torch.from_numpy(pp).to(dev); I = torch.from_numpy(ii.view(np.int64)).to(dev); W = torch.from_numpy(ww).to(dev)
    for _ in range(3): minhash_batch(P, I, W, 128, fam, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): minhash_batch(P, I, W, 128, fam, check=False)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 3
print("original", run(p, i, w), "sorted desc", run(sp, si, sw), "max nnz", nnz.max(), "mean", nnz.mean())
