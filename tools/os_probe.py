"""clock64 stamps of the one-sided pair solve (CTA 0, round 5, inner round 10) from a
-DSVDK_PROBES build: SVDK_LIB=build/exp0/libsvdk.so python tools/os_probe.py [n]."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200 import _lib  # noqa: E402
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
s = colmajor(n, n, ld=n)
s.copy_(x + x.t())
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.eig_sym(s)
    e1.record()
    torch.cuda.synchronize()
    print(f"eig n={n}: {e0.elapsed_time(e1):.2f} ms, sweeps={eng.ctx.last_sweeps()}", flush=True)
buf = (ctypes.c_longlong * 16)()
_lib.load().svdk_debug_jacobi_probe(buf)
st = list(buf)
print(f"CTA0: prologue {st[1] - st[0]}, inner rounds {st[2] - st[1]}, NS+store {st[3] - st[2]}, total {st[3] - st[0]}")
print(f"inner round 10: shuffles+dots issued {st[4]}, past barrier {st[5]}, sums landed {st[6]}, "
      f"rotation done {st[7]}, applied {st[8]}")
