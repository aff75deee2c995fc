"""clock64 stamps of one quad-scheme super-pair solve (CTA 0, round 5) at n = 4096
(development probe; needs a -DSVDK_PROBES build loaded through SVDK_LIB)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200 import _lib  # noqa: E402
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
x = torch.randn(2 * n, n, dtype=torch.float64, device="cuda")
s = colmajor(n, n, ld=n)
s.copy_(x.t() @ x)
eng.eig_sym(s)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 16)()
_lib.load().svdk_debug_jacobi_probe(buf)
t = list(buf)
print("load", t[1] - t[0], "| stage B: solve+NS", t[2] - t[1], "transform", t[3] - t[2],
      "| stage C: gather", t[4] - t[3], "solve+NS", t[5] - t[4], "transform+store", t[7] - t[5],
      "| total", t[7] - t[0], "cycles")
