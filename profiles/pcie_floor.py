"""PCIe floor for the e2e leg: pinned host -> device copy of the cfg2 input
(1.64 GB) alone, and with the 0.21 GB device -> host output copy concurrent."""
import json
import time

import torch

dev = torch.device("cuda", 0)
h_in = torch.empty(1_639_200_008 // 8, dtype=torch.int64).pin_memory()
h_out = torch.empty(205_200_000 // 8, dtype=torch.int64).pin_memory()
d_in = torch.empty_like(h_in, device=dev)
d_out = torch.empty_like(h_out, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
res = {}
for name, both in (("h2d", False), ("h2d+d2h", True)):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        if both:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    res[name] = {"ms": best * 1e3, "h2d_GBps": h_in.numel() * 8 / best / 1e9}
print(json.dumps(res))
