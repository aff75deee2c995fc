"""Small-shape exercise of every engine path, for compute-sanitizer runs."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1906_12085_b200 import svdkit as sk  # noqa: E402

rng = np.random.default_rng(0)
for m, n in ((37, 13), (130, 66), (300, 129)):
    a = np.asfortranarray(rng.standard_normal((m, n)))
    sk.gram(a)
    sk.matmul(a, rng.standard_normal((n, 7)))
    sk.matmul_transposed_left(a, rng.standard_normal((m, 5)))
    sk.qr_thin(a)
    x = rng.standard_normal((n, n))
    sk.eig_sym(x + x.T)
    s = sk.truncated_svd(a)
    sk.randomized_pca(a, sk.MethodParams(n // 2, 2, sk.RngSeed(1)))
    sk.krylov_svd(a, sk.MethodParams(4, 2, sk.RngSeed(1)))
    sk.lanczos_svd(a, 0, sk.RngSeed(1))
    sk.fit_pca(a, sk.Orientation.RowsAreExamples, sk.SvdMethod.Randomized, sk.MethodParams(n, 1, sk.RngSeed(2)))
    sk.residual_delta(a, s)
sk.qr_thin(np.zeros((20, 4)))
# Lanczos GEMV pair in every cluster size (1/2/4 CTAs exchanging y over DSMEM)
# and the device-side breakdown/restart path (rank-deficient A)
import os  # noqa: E402
b = np.asfortranarray(rng.standard_normal((300, 3)) @ rng.standard_normal((3, 40)))
for cs in ("1", "2", "4"):
    os.environ["SVDK_GEMV_CS"] = cs
    sk.lanczos_svd(np.asfortranarray(rng.standard_normal((333, 150))), 0, sk.RngSeed(3))
    sk.lanczos_svd(b, 0, sk.RngSeed(4))
os.environ.pop("SVDK_GEMV_CS")
# rank-deficient qr_thin (eigen-based basis + the small Householder QR)
h = np.asfortranarray(np.hstack([b[:, :5], b[:, :2] @ rng.standard_normal((2, 3))]))
sk.qr_thin(h)
# Lanczos tridiagonal solver, then its dense fallback
a = np.asfortranarray(rng.standard_normal((900, 200)))
sk.lanczos_svd(a, 0, sk.RngSeed(6))
os.environ["SVDK_LANCZOS_TRIDIAG"] = "0"
sk.lanczos_svd(a, 0, sk.RngSeed(6))
os.environ.pop("SVDK_LANCZOS_TRIDIAG")
# the synthetic generator (device) and the host-staged sharded path (2 ranks, threads)
import threading  # noqa: E402

import torch  # noqa: E402

from paper_1906_12085_b200 import synth  # noqa: E402
from paper_1906_12085_b200._lib import HostGroup  # noqa: E402
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402
eng = Engine(0)
a_dev = synth.device_matrix(eng, 2002, 64, np.linspace(1.0, 0.1, 64), 1e-3)
grp = HostGroup(2)
engs = [Engine(0) for _ in range(2)]
shards = []
for r, e in enumerate(engs):
    e.ctx.attach_host_group(grp, r)
    s_ = colmajor(1001, 64)
    s_.copy_(a_dev[1001 * r:1001 * (r + 1)])
    shards.append(s_)
torch.cuda.synchronize()
ths = [threading.Thread(target=lambda r=r: engs[r].pca(shards[r], method=1, l=32, q=1, seed=3))
       for r in range(2)]
[t.start() for t in ths]
[t.join() for t in ths]
print("sanitize probe done")
