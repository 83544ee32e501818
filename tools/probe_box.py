"""One-off probe of the GPU box: host cores, GPU, cuBLAS int8 (torch._int_mm) throughput.

The int8 figure is used as the measured int8 dense reference beside the
driver-written MEASURED_PEAKS.json (which only carries bf16 and HBM).
"""
import json, os, subprocess, time
import torch

out = {"nproc": os.cpu_count()}
try:
    out["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception as e:  # noqa
    out["cpu_model"] = str(e)
out["smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.max.sm,memory.total,power.limit", "--format=csv"], capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
res = {}
for n in (8192, 16384):
    a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device=dev)
    b = torch.randint(-127, 128, (n, n), dtype=torch.int8, device=dev).t().contiguous().t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    t0 = time.time(); cnt = 0
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 3:
        torch._int_mm(a, b); cnt += 1
    e1.record(); torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / 1e3 / cnt
    res[n] = {"burst_tops": 2 * n**3 / best / 1e12, "sustained_tops": 2 * n**3 / sus / 1e12}
out["cublas_int8_int_mm"] = res
# fp64 cuBLAS DGEMM for context (native FP64 the emulation competes with)
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
for _ in range(2): a @ b
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): a @ b
e1.record(); torch.cuda.synchronize()
out["cublas_dgemm_8192_tflops"] = 2 * n**3 * 5 / (e0.elapsed_time(e1) / 1e3) / 1e12
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
