"""GPU diagnostic: engine SYRK vs cuBLAS on a config's A (raw and centred)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200 import synth  # noqa: E402
from paper_1906_12085_b200.engine import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = synth.CONFIGS[name]
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
a = synth.config_device_matrix(eng, cfg)
g = eng.gram(a)
torch.cuda.synchronize()
gc = a.t() @ a
torch.cuda.synchronize()
print("raw: max|G_eng - G_cublas| / max|G|", float((g - gc).abs().max() / gc.abs().max()))
gz = np.load(f"tests/golden/{name}.npz")
mean_ref = torch.from_numpy(np.asarray(gz["mean"])).cuda()
mu = a.sum(0) / a.shape[0]
print("mean: max|mu_torch - mu_ref|", float((mu - mean_ref).abs().max()), "max|mu|", float(mu.abs().max()))
out = eng.pca(a, method=0, center=2, threshold=cfg.t)
mean_eng = out.mean
print("mean: max|mu_eng - mu_ref|", float((mean_eng - mean_ref).abs().max()))
g2 = eng.gram(a)
torch.cuda.synchronize()
gc2 = a.t() @ a
print("centred: max|G_eng - G_cublas| / max|G|", float((g2 - gc2).abs().max() / gc2.abs().max()))
w = torch.linalg.eigvalsh(gc2).flip(0).cpu().numpy()
lam = np.asarray(gz["truncated_lambda"])
print("eigvalsh(cuBLAS G of engine-centred A) vs ref", float(np.max(np.abs(w - lam) / lam)))
print("total eng", out.total, "ref", float(gz["total"]))
