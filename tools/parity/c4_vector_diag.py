"""Where does the c4 per-vector eigenvector disagreement come from? (GPU
diagnostic): engine Jacobi vs cuSOLVER eigh on the engine's own Gram, and
both vs the compiled reference's fixture."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200 import synth  # noqa: E402
from paper_1906_12085_b200.engine import Engine  # noqa: E402
from tests.parity import fixture_parity, gap_groups, topk_sine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
gz = np.load(os.path.join("tests", "golden", f"{name}.npz"))
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
cfg = synth.CONFIGS[str(gz["cfg"])]
a = synth.config_device_matrix(eng, cfg)
out = eng.pca(a, method=0, center=2, threshold=cfg.t)
sig = out.sigma[:out.rank].cpu().numpy()
vj = out.v[:, :out.rank].cpu().numpy()
g = eng.gram(a)
torch.cuda.synchronize()
gs = 0.5 * (g + g.t())
w, v = torch.linalg.eigh(gs)
w = w.flip(0).cpu().numpy()
v = v.flip(1).cpu().numpy()
res = {"jacobi_vs_ref": fixture_parity(gz, "truncated", sig * sig, vj, out.k),
       "eigh_ourG_vs_ref": fixture_parity(gz, "truncated", w, v, out.k)}
lam = np.asarray(gz["truncated_lambda"])
k = int(gz["truncated_k"])
worst = 0.0
for grp in gap_groups(lam, 1e-6):
    if len(grp) == 1 and grp[0] < k:
        worst = max(worst, topk_sine(vj[:, grp], v[:, grp]))
res["jacobi_vs_eigh_ourG_per_vector_max"] = worst
res["sweeps"] = eng.ctx.last_sweeps()
print(json.dumps(res, indent=1, default=float))
