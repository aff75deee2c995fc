"""GPU diagnostic: the engine NN GEMM of the generator (X chunk @ M, exact in
fp64) against cuBLAS, bitwise, chunk by chunk (SVDK_LIB selects a build)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200 import synth  # noqa: E402
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = synth.CONFIGS[name]
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
g = synth.device_gram_x(eng, cfg.m, cfg.n)
mix, _ = synth.mixing(g.cpu().numpy(), cfg.spectrum(), synth.MATRIX_SEED)
mdev = torch.from_numpy(np.ascontiguousarray(mix.T)).cuda().t()
chunk = 1 << 20
x = colmajor(chunk, cfg.n)
c = colmajor(chunk, cfg.n)
lib = __import__("paper_1906_12085_b200._lib", fromlist=["load"]).load()
tot = 0
for rep in range(2):
    for r0 in range(0, cfg.m, chunk):
        lib.svdk_dev_synth_fill(eng.ctx.handle, synth.MATRIX_SEED, 1, 1, cfg.m, r0, chunk, cfg.n,
                                __import__("ctypes").c_void_p(x.data_ptr()), x.stride(1))
        eng.gemm(x, mdev, c=c)
        ref = x @ mdev
        torch.cuda.synchronize()
        bad = int((c != ref).sum())
        tot += bad
        if bad:
            idx = (c != ref).nonzero()
            print(f"rep {rep} chunk {r0 // chunk}: {bad} mismatches, rows {int(idx[:, 0].min())}..{int(idx[:, 0].max())}",
                  flush=True)
print(os.environ.get("SVDK_LIB", "default"), "total mismatches", tot, flush=True)
