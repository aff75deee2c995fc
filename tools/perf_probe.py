"""Quick per-kernel timing on the GPU (development probe, not the bench)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


eng = Engine(0)
torch.cuda.set_stream(eng.stream)
res = {}
for (m, n) in [(200000, 1024), (20000, 256), (65536, 4096)]:
    a = colmajor(m, n)
    a.copy_(torch.randn(m, n, dtype=torch.float64, device="cuda"))
    ms = timeit(lambda: eng.gram(a))
    res[f"gram_{m}x{n}_tflops"] = m * n * (n + 1) / ms / 1e9
    b = colmajor(n, n)
    b.copy_(torch.randn(n, n, dtype=torch.float64, device="cuda"))
    ms = timeit(lambda: eng.gemm(a, b))
    res[f"gemm_nn_{m}x{n}x{n}_tflops"] = 2 * m * n * n / ms / 1e9
    y = colmajor(m, n)
    y.copy_(torch.randn(m, n, dtype=torch.float64, device="cuda"))
    ms = timeit(lambda: eng.gemm(a, y, transa=True))
    res[f"gemm_tn_{m}x{n}x{n}_tflops"] = 2 * m * n * n / ms / 1e9
    torch.cuda.synchronize()
    print(json.dumps(res), flush=True)
for n in (256, 1024, 2048):
    x = torch.randn(n, n, dtype=torch.float64, device="cuda")
    s = colmajor(n, n, ld=n)
    s.copy_(x + x.t())
    t0 = time.time()
    ms = timeit(lambda: eng.eig_sym(s), reps=2)
    res[f"eig_{n}_ms"] = ms
    res[f"eig_{n}_sweeps"] = eng.ctx.last_sweeps()
    print(json.dumps(res), flush=True)
