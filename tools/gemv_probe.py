"""Run a few Lanczos steps on a c3-shaped matrix (for ncu captures of gemv_pair)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 500000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
a = colmajor(m, n)
a.copy_(torch.randn(m, n, dtype=torch.float64, device="cuda"))
eng.ctx.set_timing(True)
out = eng.pca(a, method=3, l=steps, center=False, threshold=0.5)
torch.cuda.synchronize()
g = eng.ctx.timing("gemv_pair")
print(f"gemv_pair: {g['count']} launches, {g['ms'] / g['count']:.3f} ms each, "
      f"{g['bytes'] / (g['ms'] / 1e3) / 1e9 / g['count'] * g['count']:.0f} GB/s algorithmic")
