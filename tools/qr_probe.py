"""qr_thin (CholeskyQR2) on a c2-sized H: timing + per-phase breakdown."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
h = colmajor(m, p)
h.copy_(torch.randn(m, p, dtype=torch.float64, device="cuda"))
for _ in range(2):
    q, r, rank = eng.qr_thin(h)
torch.cuda.synchronize()
eng.ctx.set_timing(True)
eng.ctx.timing_reset()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(eng.stream)
q, r, rank = eng.qr_thin(h)
e1.record(eng.stream)
torch.cuda.synchronize()
print(f"qr_thin {m}x{p}: {e0.elapsed_time(e1):.2f} ms rank {rank}")
for nm in eng.ctx.timing_names():
    t = eng.ctx.timing(nm)
    print(f"  {nm}: {t['count']} launches {t['ms']:.2f} ms {t['flops'] / max(t['ms'], 1e-9) / 1e9:.1f} TF/s")
print("orth", float((q.T @ q - torch.eye(p, dtype=torch.float64, device='cuda')).abs().max()))
import ctypes
from paper_1906_12085_b200 import _lib
buf = (ctypes.c_longlong * 4)()
_lib.load().svdk_debug_chol_probe(buf)
print("chol_diag block 0 cycles: load", buf[0], "factor", buf[1], "inverse+store", buf[2])
