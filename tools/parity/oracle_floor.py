"""Noise floor of the per-vector eigenvector comparison at a full-size config
(test infrastructure / evidence, CPU): the reference fixture's eigenvectors
(reference gram in fixed row blocks + reference eig_sym, tests/golden/<cfg>.npz)
against LAPACK eigh of an independently summed Gram of the SAME centred input
(numpy/OpenBLAS in 262144-row blocks). Both are correct to rounding; their
per-vector sines show how far two correct computations of this spectrum can
disagree vector by vector, as a function of the relative gap (Davis-Kahan:
sine ~ eps_G / gap). Writes profiles/r2_<cfg>_oracle_floor.json.

    python tools/parity/oracle_floor.py c4
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1906_12085_b200 import synth  # noqa: E402
from tests.parity import gap_groups, topk_sine  # noqa: E402


def main(name):
    gz = np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz"))
    cfg = synth.CONFIGS[str(gz["cfg"])]
    m, n, seed = int(gz["m"]), int(gz["n"]), int(gz["seed"])
    mean = np.asarray(gz["mean"])
    t0 = time.time()
    mix, _ = synth.mixing(synth.host_gram_x(m, n, seed, chunk=1 << 18), cfg.spectrum(n), seed)
    g = np.zeros((n, n))
    rows = 1 << 18
    for r0 in range(0, m, rows):
        a = synth.host_matrix(m, n, cfg.spectrum(n), cfg.sigma, seed, row0=r0, rows=min(rows, m - r0), mix=mix)
        a -= mean[None, :]
        g += a.T @ a
        del a
    print("numpy gram", f"{time.time() - t0:.0f}s", flush=True)
    w, v = np.linalg.eigh(g)
    w, v = w[::-1], v[:, ::-1]
    lam_ref = np.asarray(gz["truncated_lambda"])
    k = int(gz["truncated_k"])
    vk = np.asarray(gz["truncated_vk"]) if "truncated_vk" in gz else None
    out = {"config": name, "eig_rel_err_ref_vs_eigh": float(np.max(np.abs(w[:len(lam_ref)] - lam_ref) / lam_ref)),
           "note": "reference (block gram + eig_sym) vs LAPACK eigh of a numpy-summed Gram of the same centred input"}
    if vk is not None:
        out["topK_sine"] = topk_sine(v[:, :k], vk)
        rows_out = []
        scale = lam_ref[0]
        for grp in gap_groups(lam_ref, 1e-6):
            if len(grp) != 1 or grp[0] >= k:
                continue
            i = grp[0]
            gap = min(lam_ref[i - 1] - lam_ref[i] if i > 0 else np.inf,
                      lam_ref[i] - lam_ref[i + 1] if i + 1 < len(lam_ref) else np.inf) / scale
            rows_out.append((i, gap, topk_sine(v[:, [i]], vk[:, [i]])))
        arr = np.array(rows_out)
        out["per_vector_sine_max"] = float(arr[:, 2].max())
        out["sine_times_gap_max"] = float((arr[:, 1] * arr[:, 2]).max())
        out["sine_times_gap_median"] = float(np.median(arr[:, 1] * arr[:, 2]))
        for thr in (1e-6, 2e-6, 5e-6, 1e-5, 2e-5):
            sel = arr[:, 1] >= thr
            out[f"per_vector_sine_max_gap_ge_{thr:g}"] = float(arr[sel, 2].max()) if sel.any() else 0.0
        worst = arr[np.argsort(-arr[:, 2])[:8]]
        out["worst"] = [{"index": int(a), "rel_gap": float(b), "sine": float(c)} for a, b, c in worst]
    path = os.path.join(ROOT, "profiles", f"r2_{name}_oracle_floor.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c4")
