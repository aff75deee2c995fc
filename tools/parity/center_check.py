"""GPU diagnostic: in-place centring of a config's A (svdk_dev_pca center=2)."""
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
m = a.shape[0]
blk = 1 << 17
starts = [0, m // 4, m // 2, (3 * m) // 4, m - blk]
raws = [a[s:s + blk].clone() for s in starts]
out = eng.pca(a, method=0, center=2, threshold=cfg.t)
torch.cuda.synchronize()
mu = out.mean
for s, r in zip(starts, raws):
    diff = a[s:s + blk] - (r - mu)
    bad = diff != 0
    print("rows", s, "elements differing from raw - mean:", int(bad.sum()), "of", diff.numel())
    if bad.any():
        idx = bad.nonzero()
        print("   first bad (row, col):", idx[:3].tolist(), "last:", idx[-3:].tolist())
cm = a.sum(0) / a.shape[0]
print("max |column mean after centring|", float(cm.abs().max()))
