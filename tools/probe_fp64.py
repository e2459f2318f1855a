"""Measuring-stick probe (not part of the engine): device properties, cuBLAS
DGEMM throughput (burst and sustained) and fp64 copy bandwidth.  cuBLAS is
used here only as the FP64 roofline denominator, never by the engine."""
import json, time, torch
p = torch.cuda.get_device_properties(0)
out = {"name": p.name, "sms": p.multi_processor_count, "l2_bytes": getattr(p, "L2_cache_size", None),
       "total_mem": p.total_memory, "cc": [p.major, p.minor]}
def bench(fn, iters):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / iters * 1e-3
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a); c = torch.empty_like(a)
    for _ in range(3): torch.matmul(a, b, out=c)
    t = min(bench(lambda: torch.matmul(a, b, out=c), 5) for _ in range(3))
    out[f"dgemm_tflops_{n}"] = 2 * n**3 / t / 1e12
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a); c = torch.empty_like(a)
t0 = time.time(); cnt = 0
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); s.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b, out=c); cnt += 1
    if cnt % 8 == 0: torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
out["dgemm_tflops_sustained_8192"] = 2 * n**3 * cnt / (s.elapsed_time(e) * 1e-3) / 1e12
x = torch.empty(2**27, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
t = min(bench(lambda: y.copy_(x), 10) for _ in range(3))
out["copy_gbs_fp64_1GiB"] = 2 * x.numel() * 8 / t / 1e9
print(json.dumps(out))
json.dump(out, open("gpurun_out/probe_fp64.json", "w"), indent=1)
