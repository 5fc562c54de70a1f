"""Dev tool: cost of page-locking a pageable host array in place
(cudaHostRegister) and the DMA rate from it, against the staged copy."""
import ctypes
import time
import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so.12") if False else None
torch.cuda.init()
rt = torch.cuda.cudart()
for mb in (116, 464):
    n = mb << 20
    src = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    for rep in range(2):
        t0 = time.perf_counter()
        r = rt.cudaHostRegister(src.ctypes.data, n, 0)
        t1 = time.perf_counter()
        dev.copy_(torch.from_numpy(src), non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rt.cudaHostUnregister(src.ctypes.data)
        t3 = time.perf_counter()
        print(f"{mb} MB: register {1e3 * (t1 - t0):.2f} ms (rc {r}), DMA {1e3 * (t2 - t1):.2f} ms "
              f"({n / (t2 - t1) / 1e9:.1f} GB/s), unregister {1e3 * (t3 - t2):.2f} ms")
