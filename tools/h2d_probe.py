import torch, time
n = 64 * 1024 * 1024  # 512 MB of float64
a = torch.empty(n, dtype=torch.float64).pin_memory()
b = torch.empty(n, dtype=torch.float64).pin_memory()
da = torch.empty(n, dtype=torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1):
        da.copy_(a, non_blocking=True); db.copy_(b, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        da.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2):
        db.copy_(b, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        a.copy_(da, non_blocking=True)
    with torch.cuda.stream(s2):
        db.copy_(b, non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter() - t
    print(f"1 stream {2*n*8/t1/1e9:.1f} GB/s, 2 streams {2*n*8/t2/1e9:.1f} GB/s, duplex {2*n*8/t3/1e9:.1f} GB/s")
