import time, numpy as np, torch, ctypes
a = np.random.default_rng(0).random(205_000_000)  # 1.64 GB
cudart = torch.cuda.cudart()
torch.cuda.init()
for it in range(2):
    t = time.perf_counter()
    r = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    r2 = cudart.cudaHostUnregister(a.ctypes.data)
    t2 = time.perf_counter()
    print("register", r, (t1 - t) * 1e3, "ms; unregister", r2, (t2 - t1) * 1e3, "ms")
