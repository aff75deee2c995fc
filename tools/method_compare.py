"""BASELINE.json configs[4] ("full-spectrum method comparison"): all n
eigenpairs of the c5 matrix (65536 x 4096, s_i = 1/(1 + 0.01 i), noise 1e-2,
column-centred) by truncated SVD (Gram + Jacobi), randomized PCA (l = min(k + p,
n) = n, p = 10, q = 3, CholeskyQR2) and Lanczos (n steps, full
reorthogonalisation), each timed on the device (CUDA events, A resident,
centring inside the step) and compared with the truncated result: eigenvalue
relative error, top-K subspace sine (complement-based, never sqrt(1 - cos^2)),
K at t = 0.90. The compiled reference needs hours per method at this size
(SURVEY 7), so agreement is reported against the engine's Gram route, which
the parity tests pin to the reference at c1 and c2mid.

  python tools/method_compare.py [config] [--reps R] > profiles/r1_c5_methods.json
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c5")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    m, n, t = cfg["m"], cfg["n"], cfg["t"]
    eng = Engine(0)
    torch.cuda.set_stream(eng.stream)
    A0 = bench.generate(cfg, m, torch.device("cuda", 0), 0)
    A = colmajor(m, n)
    methods = [("truncated", 0, 0, 0), ("randomized", 1, min(n + 10, n), 3), ("lanczos", 3, 0, 0)]
    res = {"config": cfg["desc"], "m": m, "n": n, "threshold": t, "methods": {}}
    outs = {}
    for name, mid, l, q in methods:
        best = None
        for _ in range(args.reps):
            A.copy_(A0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
            o = eng.pca(A, method=mid, l=l, q=q, seed=4242, center=2, threshold=t)
            e1.record(eng.stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        outs[name] = (o.sigma[:o.rank].clone() ** 2, o.v[:, :o.rank].clone(), o.k, o.rank)
        res["methods"][name] = {"ms": round(best, 2), "rows_per_s": m / (best / 1e3), "K": o.k, "rank": o.rank,
                                "params": {"l": l, "q": q} if mid == 1 else ({"steps": n} if mid == 3 else {})}
        print(json.dumps({name: res["methods"][name]}), file=sys.stderr, flush=True)
    lam_t, v_t, k_t, _ = outs["truncated"]
    for name in ("randomized", "lanczos"):
        lam, v, k, rank = outs[name]
        r = min(rank, lam_t.numel())
        rel = float(((lam[:r] - lam_t[:r]).abs() / lam_t[:r]).max())
        kk = k_t
        # || (I - V V^T) V_t ||_2 on the top-K subspaces
        vk, vt = v[:, :kk], v_t[:, :kk]
        resid = vt - vk @ (vk.T @ vt)
        sine = float(torch.linalg.matrix_norm(resid, ord=2))
        res["methods"][name].update({"eig_rel_err_vs_truncated": rel, "topK_subspace_sine_vs_truncated": sine,
                                     "K_matches_truncated": k == k_t})
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
