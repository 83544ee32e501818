"""cudaHostRegister / cudaHostUnregister cost on pageable numpy buffers (development probe)."""
import time, numpy as np, torch
cr = torch.cuda.cudart()
torch.cuda.init()
for mb in (64, 512, 1024):
    a = np.ones(mb * 131072)  # mb MiB
    ptr = a.ctypes.data
    for rep in range(3):
        t0 = time.perf_counter()
        r = cr.cudaHostRegister(ptr, a.nbytes, 0)
        t1 = time.perf_counter()
        r2 = cr.cudaHostUnregister(ptr)
        t2 = time.perf_counter()
        print(mb, "MiB register", round((t1 - t0) * 1e3, 2), "ms unregister", round((t2 - t1) * 1e3, 2), "ms", r, r2)
