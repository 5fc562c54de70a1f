"""Dev tool: host->device copy paths on the GPU box (pageable via the driver,
pinned DMA, host memcpy into pinned buffers with N threads)."""
import os
import time
import threading
import numpy as np
import torch

n = 464 << 20
src = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
pin = torch.empty(n, dtype=torch.uint8).pin_memory()
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for rep in range(2):
    t = time.perf_counter(); dev.copy_(torch.from_numpy(src)); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"pageable H2D (driver): {n / dt / 1e9:.1f} GB/s")
    t = time.perf_counter(); dev.copy_(pin, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"pinned H2D: {n / dt / 1e9:.1f} GB/s")
    pn = pin.numpy()
    for nth in (1, 4, 8, 16, 32):
        def work(i):
            a, b = n * i // nth, n * (i + 1) // nth
            pn[a:b] = src[a:b]
        t = time.perf_counter()
        ths = [threading.Thread(target=work, args=(i,)) for i in range(nth)]
        [x.start() for x in ths]; [x.join() for x in ths]
        dt = time.perf_counter() - t
        print(f"host memcpy pageable->pinned, {nth} threads: {n / dt / 1e9:.1f} GB/s")
