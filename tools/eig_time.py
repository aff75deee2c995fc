"""Time eig_sym on random symmetric matrices (development probe, not the bench)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

eng = Engine(0)
torch.cuda.set_stream(eng.stream)
res = {}
for n in [int(x) for x in (sys.argv[1:] or ["256", "1024", "2048", "4096"])]:
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randn(2 * n, n, dtype=torch.float64, device="cuda", generator=g)
    s = colmajor(n, n, ld=n)
    s.copy_(x.t() @ x)  # SPD Gram-like spectrum
    eng.eig_sym(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(2 if n >= 4096 else 3):
        e0.record()
        w, v = eng.eig_sym(s)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    ref = torch.linalg.eigvalsh(s).flip(0)
    res[n] = {"ms": round(best, 3), "sweeps": eng.ctx.last_sweeps(),
              "eig_err": float((w - ref).abs().max() / ref.abs().max())}
    print(json.dumps(res), flush=True)
