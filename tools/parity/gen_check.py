"""GPU diagnostic: the device generator's rows vs the host generator at many
random rows of a config (exactness of X M through the engine GEMM)."""
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
g = synth.device_gram_x(eng, cfg.m, cfg.n)
mix, _ = synth.mixing(g.cpu().numpy(), cfg.spectrum(), synth.MATRIX_SEED)
a = synth.device_rows(eng, mix, cfg.m, cfg.n, cfg.sigma)
bad = 0
full = len(sys.argv) > 2 and sys.argv[2] == "full"
blocks = range(0, cfg.m, 1 << 18) if full else sorted(np.random.default_rng(1).integers(0, cfg.m - 64, 40).tolist())
for r0 in blocks:
    rows = min(1 << 18, cfg.m - r0) if full else 64
    host = synth.host_matrix(cfg.m, cfg.n, cfg.spectrum(), cfg.sigma, row0=r0, rows=rows, mix=mix)
    dev = a[r0:r0 + rows].cpu().numpy()
    if not np.array_equal(host, dev):
        d = np.argwhere(host != dev)
        bad += 1
        print("MISMATCH rows", r0, "n_diff", len(d), "first", d[:4].tolist(), "maxabs", np.max(np.abs(host - dev)),
              flush=True)
print("checked", len(blocks), "blocks; bad blocks:", bad, flush=True)
# an NN GEMM of the same shape class against cuBLAS
x = torch.randn(200000, 1024, dtype=torch.float64, device="cuda")
from paper_1906_12085_b200.engine import colmajor  # noqa: E402
xa = colmajor(200000, 1024)
xa.copy_(x)
m_ = torch.from_numpy(np.ascontiguousarray(mix.T)).cuda().t()
c = eng.gemm(xa, m_)
torch.cuda.synchronize()
ref = xa @ m_
print("NN vs cuBLAS max rel", float((c - ref).abs().max() / ref.abs().max()))
