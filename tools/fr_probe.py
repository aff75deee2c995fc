"""clock64 stamps of the fused round kernel (solve CTA 0 and worker CTA 0, round 5) from a
-DSVDK_PROBES build: SVDK_LIB=build/exp0/libsvdk.so python tools/fr_probe.py [n]."""
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
for cap in (30, 3):  # the second call stops after 3 sweeps, so the stamps come from a working round
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    try:
        eng.eig_sym(s, cap)
    except Exception:  # noqa: BLE001
        pass
    e1.record()
    torch.cuda.synchronize()
    print(f"eig n={n} cap={cap}: {e0.elapsed_time(e1):.2f} ms, sweeps={eng.ctx.last_sweeps()}", flush=True)
buf = (ctypes.c_longlong * 16)()
_lib.load().svdk_debug_jacobi_probe(buf)
st = list(buf)
print(f"solve CTA0: before wait {st[1] - st[0]}, prologue {st[2] - st[1]}, rounds {st[3] - st[2]}, "
      f"norm+store {st[4] - st[3]}, total {st[4] - st[0]}")
print(f"worker CTA0 warp0: before wait {st[9] - st[8]}, first task {st[10] - st[9]}, all tasks {st[11] - st[9]}")
