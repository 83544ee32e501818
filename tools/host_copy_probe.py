"""Host memory bandwidth for the pageable staging path (development tool):
pageable -> pinned copies of 1 GiB with 1..16 threads, alone and while a
pinned 1 GiB H2D DMA runs.

Usage: python tools/host_copy_probe.py
"""
import concurrent.futures as cf
import json
import time

import numpy as np
import torch


def copy_threads(dst, src, nt):
    rows = src.shape[0]
    parts = [(rows * i // nt, rows * (i + 1) // nt) for i in range(nt)]
    with cf.ThreadPoolExecutor(nt) as ex:
        list(ex.map(lambda p: np.copyto(dst[p[0]:p[1]], src[p[0]:p[1]]), parts))


def main():
    n = 1 << 27  # 1 GiB of doubles
    src = np.random.default_rng(0).random((8192, n // 8192))
    dst = torch.empty(src.shape, dtype=torch.float64).pin_memory().numpy()
    h2d_src = torch.empty(src.shape, dtype=torch.float64).pin_memory()
    dev = torch.empty(src.shape, dtype=torch.float64, device="cuda")
    out = {}
    for nt in (1, 4, 8, 16):
        copy_threads(dst, src, nt)
        t = time.perf_counter()
        copy_threads(dst, src, nt)
        out[f"copy_{nt}t_GBps"] = 8 * n / (time.perf_counter() - t) / 1e9
    s = torch.cuda.Stream()
    dev.copy_(h2d_src, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s):
        dev.copy_(h2d_src, non_blocking=True)
    s.synchronize()
    out["h2d_alone_GBps"] = 8 * n / (time.perf_counter() - t) / 1e9
    t = time.perf_counter()
    with torch.cuda.stream(s):
        dev.copy_(h2d_src, non_blocking=True)
    copy_threads(dst, src, 16)
    tc = time.perf_counter() - t
    s.synchronize()
    tb = time.perf_counter() - t
    out["concurrent_copy16_GBps"] = 8 * n / tc / 1e9
    out["concurrent_both_done_s"] = tb
    print(json.dumps(out))


if __name__ == "__main__":
    main()
