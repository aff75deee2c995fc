"""Probe: cuBLAS DGEMM (torch.matmul fp64) throughput — the measured FP64 roofline denominator."""
import json, time, torch
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for N in (4096, 8192):
    a = torch.randn(N, N, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"dgemm_{N}_burst_tflops"] = 2 * N**3 / best / 1e9
# sustained 4 s
N = 8192
a = torch.randn(N, N, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
t0 = time.time(); n = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4:
    for _ in range(4): a @ b; n += 1
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
res["dgemm_8192_sustained_tflops"] = 2 * N**3 * n / e0.elapsed_time(e1) / 1e9
# tall-skinny gram like c2
A = torch.randn(200000, 1024, dtype=torch.float64, device="cuda")
for _ in range(3): A.T @ A
torch.cuda.synchronize()
e0.record()
for _ in range(5): A.T @ A
e1.record(); torch.cuda.synchronize()
res["cublas_gram_c2_tflops_2mn2"] = 2 * 200000 * 1024**2 * 5 / e0.elapsed_time(e1) / 1e9
print(json.dumps(res))
