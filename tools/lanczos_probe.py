"""Lanczos phase breakdown on a bench config (development probe, not the bench):
one warm run, then one run with the engine's per-phase CUDA-event timing.
  python tools/lanczos_probe.py [config] [method]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
method = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = dict(bench.CONFIGS[name])
m, n = cfg["m"], cfg["n"]
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
A0 = bench.generate(cfg, m, torch.device("cuda", 0), 0)
A = colmajor(m, n)
res = {}
for rep in range(2):
    A.copy_(A0)
    if rep == 1:
        eng.ctx.set_timing(True)
        eng.ctx.timing_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = eng.pca(A, method=method, l=min(n + 10, n) if method == 1 else 0, q=3 if method == 1 else 0,
                  seed=7, center=2, threshold=cfg["t"])
    e1.record()
    torch.cuda.synchronize()
    res[f"rep{rep}_ms"] = round(e0.elapsed_time(e1), 2)
res["K"] = out.k
res["phases_ms"] = {k: round(eng.ctx.timing(k)["ms"], 2) for k in eng.ctx.timing_names()}
print(json.dumps(res))
