"""GPU diagnostic for the LDS + fast-epilogue mismatch: in a wrong tile, is
the error one k-stage (16 columns of K) missing / doubled / swapped?"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200 import _lib, synth  # noqa: E402
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

cfg = synth.CONFIGS["c4"]
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
n = cfg.n
mdev = torch.randn(n, n, dtype=torch.float64, device="cuda")
mq = torch.round(mdev * 2 ** 20) / 2 ** 20  # exact products with the quantised X
m_ = colmajor(n, n)
m_.copy_(mq)
chunk = 1 << 20
x = colmajor(chunk, n)
c = colmajor(chunk, n)
lib = _lib.load()
for trial in range(6):
    lib.svdk_dev_synth_fill(eng.ctx.handle, 42, 1, 1, cfg.m, trial * chunk, chunk, n, ctypes.c_void_p(x.data_ptr()),
                            x.stride(1))
    eng.gemm(x, m_, c=c)
    ref = x @ m_
    torch.cuda.synchronize()
    bad = (c != ref)
    if not bad.any():
        print("trial", trial, "ok")
        continue
    idx = bad.nonzero()
    ti = (idx[:, 0] // 128).unique().tolist()
    tj = (idx[:, 1] // 128).unique().tolist()
    print("trial", trial, "bad elems", int(bad.sum()), "tile rows", ti[:8], "tile cols", tj[:8])
    r0, c0 = int(idx[0, 0]) // 128 * 128, int(idx[0, 1]) // 128 * 128
    tiles = {}
    for rr, cc in idx.tolist():
        tiles[(rr // 128, cc // 128)] = tiles.get((rr // 128, cc // 128), 0) + 1
    print("  bad tiles (ti, tj): count", sorted(tiles.items())[:12])
    d = (c - ref)[r0:r0 + 128, c0:c0 + 128]
    print("  bad in tile:", int((d != 0).sum()), "rows with bad:", int(((d != 0).any(1)).sum()),
          "cols with bad:", int(((d != 0).any(0)).sum()))
    best = []
    for j in range(n // 16):
        s = x[r0:r0 + 128, 16 * j:16 * j + 16] @ m_[16 * j:16 * j + 16, c0:c0 + 128]
        for sgn in (1, -1):
            e = float((d - sgn * s).abs().max())
            best.append((e, j, sgn))
    # the last k4 steps of the last stage (a too-early accumulator read)
    for q in range(1, 17):
        s = x[r0:r0 + 128, n - q:n] @ m_[n - q:n, c0:c0 + 128]
        mask = d != 0
        e = float((d[mask] + s[mask]).abs().max()) if mask.any() else 0.0
        best.append((e, f"missing last {q} k", -1))
    best.sort(key=lambda t: t[0])
    print("  closest single-stage explanation (maxabs residual, stage, sign):", best[:3],
          "max|d|", float(d.abs().max()))
