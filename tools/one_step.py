"""One device-resident fit_pca step of a bench config between cudaProfilerStart/Stop
(for `ncu --profile-from-start off` launch lists of exactly one step).
  python tools/one_step.py [config]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1906_12085_b200 import synth  # noqa: E402
from paper_1906_12085_b200.engine import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = bench.config(name)
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
A, _ = bench.generate(eng, cfg, 1, 0)
mid = bench.METHOD_ID[cfg["method"]]


def step(out=None):
    return eng.pca(A, method=mid, l=cfg["l"], q=cfg["q"], seed=synth.METHOD_SEED, center=2, threshold=cfg["t"],
                   out=out)


out = step()
out = step(out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
out = step(out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("K", out.k, "rank", out.rank)
