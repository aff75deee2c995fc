"""globaltimer stamps of the fused round kernels (rounds 1..15 of the last sweep run) from a
-DSVDK_PROBES build: SVDK_LIB=build/exp0/libsvdk.so python tools/fr_timeline.py [n]."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200 import _lib  # noqa: E402
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
s = colmajor(n, n, ld=n)
s.copy_(x + x.t())
for cap in (30, 3):
    try:
        eng.eig_sym(s, cap)
    except Exception:  # noqa: BLE001
        pass
    torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 128)()
_lib.load().svdk_debug_jacobi_timeline(buf)
t = [list(buf[8 * r:8 * r + 8]) for r in range(16)]
base = t[1][0]
print("round | solve: start  waited  end | worker0: start  waited  end | last worker end   (us, relative to round 1's solve start)")
for r in range(1, min(15, n // 16 - 1)):
    v = [(x - base) / 1e3 if x else float("nan") for x in t[r][:7]]
    print(f"{r:5d} | {v[0]:8.2f} {v[1]:8.2f} {v[2]:8.2f} | {v[3]:8.2f} {v[4]:8.2f} {v[5]:8.2f} | {v[6]:8.2f}")
