"""BASELINE.json configs[4] ("full-spectrum method comparison"): all n eigenpairs of the c5 matrix
(65536 x 4096, s_i = 1/(1 + 0.01 i), noise 1e-2, column-centred) by truncated SVD (Gram + Jacobi),
randomized PCA (l = min(k + p, n) = n, p = 10, q = 3, CholeskyQR2) and Lanczos (n steps, full
reorthogonalisation), each timed on the device (CUDA events, A resident, centring inside the step)
and compared with the ORACLE: the golden fixture tests/golden/<config>.npz computed by the compiled
reference on the same input bytes (reference gram on row blocks + reference eig_sym) —
eigenvalue relative error, K at t = 0.90, top-K subspace sine, per-vector sines.

  python tools/method_compare.py [config] [--reps R] > profiles/r2_c5_methods.json
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1906_12085_b200 import synth  # noqa: E402
from paper_1906_12085_b200.engine import Engine  # noqa: E402
from tests.parity import fixture_parity, parity_ok  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c5")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--fixture", default=None, help="fixture name under tests/golden (default: the config's)")
    args = ap.parse_args()
    cfg = bench.config(args.config)
    m, n, t = cfg["m"], cfg["n"], cfg["t"]
    gz = np.load(os.path.join(ROOT, "tests", "golden", f"{args.fixture or args.config}.npz"))
    eng = Engine(0)
    torch.cuda.set_stream(eng.stream)
    a0, _ = bench.generate(eng, cfg, 1, 0)
    a = torch.empty_like(a0)
    methods = [("truncated", 0, 0, 0), ("randomized", 1, min(n + 10, n), 3), ("lanczos", 3, 0, 0)]
    res = {"config": cfg["desc"], "m": m, "n": n, "threshold": t, "oracle": str(gz["oracle"]), "methods": {}}
    for name, mid, l, q in methods:
        best, o = None, None
        for _ in range(args.reps):
            a.copy_(a0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
            o = eng.pca(a, method=mid, l=l, q=q, seed=synth.METHOD_SEED, center=2, threshold=t)
            e1.record(eng.stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        sigma = o.sigma[:o.rank].cpu().numpy()
        p = fixture_parity(gz, "truncated", sigma * sigma, o.v[:, :o.rank].cpu().numpy(), o.k)
        res["methods"][name] = {"ms": round(best, 2), "rows_per_s": m / (best / 1e3), "K": o.k, "rank": o.rank,
                                "params": {"l": l, "q": q} if mid == 1 else ({"steps": n} if mid == 3 else {}),
                                "vs_oracle": p, "parity_ok": bool(parity_ok(p))}
        print(json.dumps({name: res["methods"][name]}, default=float), file=sys.stderr, flush=True)
    print(json.dumps(res, default=float), flush=True)


if __name__ == "__main__":
    main()
