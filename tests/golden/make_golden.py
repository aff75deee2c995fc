"""Generate the golden fixtures from the COMPILED REFERENCE (oracle/_ref).

Run here (where /root/reference exists): python tests/golden/make_golden.py [small|c1|mid]
Inputs come from tests/datagen.py (deterministic, regenerable on the GPU box);
outputs are what the unmodified reference computes on those bytes.
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Oracle  # noqa: E402
from tests.datagen import THRESHOLD, make_matrix  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).hexdigest()


def small(ref):
    m, n, seed = 300, 24, 7
    a = make_matrix(m, n, "c1", seed=seed)
    l, q, kl, ki, rseed = 24, 2, 8, 2, 1234
    t = ref.truncated_svd(a)
    r = ref.randomized_pca(a, l, q, rseed)
    k = ref.krylov_svd(a, kl, ki, rseed)
    g = ref.gram(a)
    w, v = ref.eig_sym(g)
    np.savez_compressed(os.path.join(OUT, "small.npz"), m=m, n=n, seed=seed, a=a, l=l, q=q, kl=kl, ki=ki,
                        rseed=rseed, trunc_sigma=t.sigma, trunc_u=t.u, trunc_v=t.v, rand_sigma=r.sigma,
                        rand_u=r.u, rand_v=r.v, kry_sigma=k.sigma, kry_u=k.u, kry_v=k.v, gram=g, eig_w=w,
                        eig_v=v)


def full(ref, name, cfg, m, n, seed, methods, vcols):
    t0 = time.time()
    a = make_matrix(m, n, cfg, seed=seed)
    print(name, "generated", a.shape, f"{time.time() - t0:.1f}s", flush=True)
    out = dict(m=m, n=n, seed=seed, cfg=cfg, sha256=sha(a), threshold=THRESHOLD[cfg])
    c, mean = ref.center(a, 1)
    total = ref.frobenius_norm_sq(c)
    out["total"] = total
    for meth, (l, q, rs) in methods.items():
        t0 = time.time()
        if meth == "truncated":
            s = ref.truncated_svd(c)
        elif meth == "randomized":
            s = ref.randomized_pca(c, l, q, rs)
        else:
            s = ref.krylov_svd(c, l, q, rs)
        lam = s.sigma ** 2
        out[f"{meth}_lambda"] = lam
        out[f"{meth}_v"] = s.v[:, :vcols]
        out[f"{meth}_k"] = ref.select_components(lam, total, THRESHOLD[cfg]) or 0
        out[f"{meth}_params"] = np.array([l, q, rs])
        print(name, meth, f"{time.time() - t0:.1f}s K={out[f'{meth}_k']}", flush=True)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)


if __name__ == "__main__":
    ref = Oracle("ref")
    which = sys.argv[1:] or ["small", "c1"]
    if "small" in which:
        small(ref)
    if "c1" in which:
        full(ref, "c1", "c1", 20000, 256, 42,
             {"truncated": (0, 0, 0), "randomized": (256, 2, 4242), "krylov": (128, 1, 4242)}, 256)
    if "mid" in which:
        # c2's spectrum and method at a CPU-feasible height (the full 200000 rows take ~1 h on the reference)
        full(ref, "c2mid", "c2", 20000, 1024, 42,
             {"truncated": (0, 0, 0), "randomized": (1024, 2, 4242)}, 64)
