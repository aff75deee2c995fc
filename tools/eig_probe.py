"""Run one eig_sym(n) on the GPU (for ncu launch lists / timing)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
eng = Engine(0)

torch.cuda.set_stream(eng.stream)
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
s = colmajor(n, n, ld=n)
s.copy_(x + x.t())
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    w, v = eng.eig_sym(s)
    e1.record()
    torch.cuda.synchronize()
    print(f"eig n={n}: {e0.elapsed_time(e1):.2f} ms, sweeps={eng.ctx.last_sweeps()}", flush=True)
ref = torch.linalg.eigvalsh(s.contiguous()).flip(0)
import ctypes
from paper_1906_12085_b200 import _lib
buf = (ctypes.c_longlong * 16)()
_lib.load().svdk_debug_jacobi_probe(buf)
st = list(buf)
print("pair_solve CTA0 cycles: load", st[1] - st[0], "rounds", st[2] - st[1], "| round10 lookahead: to-barrier", st[6], "(entries", st[3], "rotation", st[4], ") barrier", st[7])
print("max |dw| / ||S||_F =", float((w - ref).abs().max() / torch.linalg.norm(s)))
