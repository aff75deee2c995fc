"""One eig_sym(n) on a Gram-like matrix between cudaProfilerStart/Stop (ncu launch lists)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
g = torch.Generator(device="cuda").manual_seed(n)
x = torch.randn(2 * n, n, dtype=torch.float64, device="cuda", generator=g)
s = colmajor(n, n, ld=n)
s.copy_(x.t() @ x)
eng.eig_sym(s)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.eig_sym(s)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("sweeps", eng.ctx.last_sweeps())
