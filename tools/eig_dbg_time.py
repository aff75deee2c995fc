"""Timing-only: ms per sweep of eig_sym(n) under SVDK_JACOBI_DBG switches (results may be wrong /
the call may end in NumericalError after the sweep cap)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

eng = Engine(0)
torch.cuda.set_stream(eng.stream)
for n in [int(x) for x in sys.argv[1:]]:
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randn(2 * n, n, dtype=torch.float64, device="cuda", generator=g)
    s = colmajor(n, n, ld=n)
    s.copy_(x.t() @ x)
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        try:
            eng.eig_sym(s)
        except Exception as ex:  # noqa: BLE001
            pass
        e1.record()
        torch.cuda.synchronize()
    sw = eng.ctx.last_sweeps()
    ms = e0.elapsed_time(e1)
    print(f"n={n}: {ms:.2f} ms, {sw} sweeps, {ms / max(sw, 1):.3f} ms/sweep, "
          f"{1e3 * ms / max(sw, 1) / (n // 16):.2f} us per block round", flush=True)
