"""One NN GEMM (U = A V shape of c4, 2^20 rows) and one TN GEMM of the same
operand for ncu (development probe: `ncu -k regex:gemm_kernel -c 2 ...`)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
a = colmajor(m, n)
a.copy_(torch.randn(m, n, dtype=torch.float64, device="cuda"))
v = colmajor(n, n)
v.copy_(torch.randn(n, n, dtype=torch.float64, device="cuda"))
u = colmajor(m, n)
eng.gemm(a, v, c=u)          # NN: gemm_kernel<1>
eng.gemm(a, u, transa=True)  # TN: gemm_kernel<0>
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("nn", lambda: eng.gemm(a, v, c=u)), ("tn", lambda: eng.gemm(a, u, transa=True)),
                 ("gram", lambda: eng.gram(a))):
    best = 1e9
    for _ in range(3):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    fl = 2.0 * m * n * n if name != "gram" else 1.0 * m * n * (n + 1)
    print(f"{name}: {best:.3f} ms  {fl / best / 1e9:.2f} TF/s", flush=True)
