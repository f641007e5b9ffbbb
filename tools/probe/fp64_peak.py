"""Probe: cuBLAS DGEMM burst/sustained FP64 throughput on this B200 (roofline denominator)."""
import json, subprocess, time, torch
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"dgemm_{n}_burst_tflops"] = 2 * n**3 / best / 1e9
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader", "-lms", "200"], stdout=subprocess.PIPE, text=True)
torch.cuda.synchronize(); t0 = time.time(); k = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; k += 1
    if k % 4 == 0: torch.cuda.synchronize()
e1.record(); e1.synchronize()
smi.terminate(); lines = smi.communicate()[0].strip().splitlines()
res["dgemm_8192_sustained_tflops"] = 2 * n**3 * k / e0.elapsed_time(e1) / 1e9
res["clocks_samples"] = lines[-8:]
x = torch.empty(2 * 1024**3 // 8, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); best = 1e9
for _ in range(10):
    e0.record(); y.copy_(x); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
res["copy_gbs"] = 2 * x.numel() * 8 / best / 1e6
print(json.dumps(res, indent=1))
