"""Parity metrics — test infrastructure.

Sines are computed from the orthogonal complement, ||(I - V V^T) V_ref||_2,
never as sqrt(1 - cos^2) (which cannot resolve anything below ~1e-8).
"""
from __future__ import annotations

import numpy as np


def eig_rel_err(w, w_ref) -> float:
    w, w_ref = np.asarray(w), np.asarray(w_ref)
    assert w.shape == w_ref.shape, (w.shape, w_ref.shape)
    scale = np.maximum(np.abs(w_ref), 1e-300)
    return float(np.max(np.abs(w - w_ref) / scale)) if w.size else 0.0


def subspace_sine(v, v_ref) -> float:
    """||(I - V V^T) V_ref||_2 for orthonormal V, V_ref (same column count)."""
    v, v_ref = np.asarray(v), np.asarray(v_ref)
    if v_ref.shape[1] == 0:
        return 0.0
    r = v_ref - v @ (v.T @ v_ref)
    return float(np.linalg.norm(r, 2))


def gap_groups(w, rel_gap=1e-6):
    """Indices grouped into clusters whose neighbouring relative gap < rel_gap."""
    w = np.asarray(w)
    scale = max(abs(w[0]), 1e-300)
    groups, cur = [], [0]
    for i in range(1, len(w)):
        if (w[i - 1] - w[i]) / scale < rel_gap:
            cur.append(i)
        else:
            groups.append(cur)
            cur = [i]
    groups.append(cur)
    return groups


def per_vector_sines(v, w_ref, v_ref, rel_gap=1e-6):
    """Max sine over gap-separated vectors and over cluster subspaces."""
    worst_single, worst_cluster = 0.0, 0.0
    for g in gap_groups(w_ref, rel_gap):
        s = subspace_sine(v[:, g], v_ref[:, g])
        if len(g) == 1:
            worst_single = max(worst_single, s)
        else:
            worst_cluster = max(worst_cluster, s)
    return worst_single, worst_cluster


def orthogonality(v) -> float:
    v = np.asarray(v)
    return float(np.max(np.abs(v.T @ v - np.eye(v.shape[1])))) if v.shape[1] else 0.0


def spectral_norm(r) -> float:
    """||r||_2 through the smaller Gram side (fast for tall-skinny r)."""
    r = np.asarray(r)
    if r.size == 0:
        return 0.0
    g = r.T @ r if r.shape[0] >= r.shape[1] else r @ r.T
    return float(np.sqrt(max(np.linalg.eigvalsh(g)[-1], 0.0)))


def topk_sine(v_k, v_ref_k) -> float:
    """||(I - V V^T) V_ref||_2 for the top-K bases (same column count)."""
    v_k, v_ref_k = np.asarray(v_k), np.asarray(v_ref_k)
    return spectral_norm(v_ref_k - v_k @ (v_k.T @ v_ref_k))


def fixture_parity(gz, prefix, lam, basis, k, rel_gap=1e-6) -> dict:
    """Compare an engine result (eigenvalues lam, basis n x >=K, selected K)
    with a golden fixture written by tests/golden/make_golden.py (SURVEY §8c bars):
    eigenvalue relative error, K vs K_ref, the top-K subspace sine and the worst
    per-vector sine over gap-separated vectors (clusters as subspaces)."""
    lam_ref = np.asarray(gz[f"{prefix}_lambda"])
    k_ref = int(gz[f"{prefix}_k"])
    lam = np.asarray(lam)
    basis = np.asarray(basis)
    out = {"K": int(k) if k is not None else None, "K_ref": k_ref,
           "eig_rel_err": eig_rel_err(lam[:len(lam_ref)], lam_ref) if len(lam) >= len(lam_ref) else float("inf")}
    vk = basis[:, :k_ref]
    groups = [g for g in gap_groups(lam_ref, rel_gap) if g[-1] < k_ref]
    if f"{prefix}_v" in gz or f"{prefix}_vk" in gz:
        ref_k = np.asarray(gz[f"{prefix}_v"])[:, :k_ref] if f"{prefix}_v" in gz else np.asarray(gz[f"{prefix}_vk"])
        out["topK_sine"] = topk_sine(vk, ref_k)
        single = cluster = 0.0
        worst = (0.0, -1, 0.0)
        sg = 0.0
        scale = max(abs(lam_ref[0]), 1e-300)
        for g in groups:
            s = topk_sine(basis[:, g], ref_k[:, g])
            if len(g) == 1:
                single = max(single, s)
                i = g[0]
                gap = min(lam_ref[i - 1] - lam_ref[i] if i > 0 else np.inf,
                          lam_ref[i] - lam_ref[i + 1] if i + 1 < len(lam_ref) else np.inf) / scale
                sg = max(sg, s * gap)
                if s > worst[0]:
                    worst = (s, i, gap)
            else:
                cluster = max(cluster, s)
        out["per_vector_sine"], out["cluster_sine"] = single, cluster
        out["per_vector_worst"] = {"sine": worst[0], "index": worst[1], "rel_gap": worst[2]}
        out["sine_times_gap_max"] = sg
        out["vectors_checked"] = int(sum(len(g) for g in groups))
    else:
        vperp = np.asarray(gz[f"{prefix}_vperp"])
        out["topK_sine"] = spectral_norm(vk.T @ vperp)
        if f"{prefix}_vidx" in gz:
            idx = np.asarray(gz[f"{prefix}_vidx"])
            vs = np.asarray(gz[f"{prefix}_vsample"])
            out["per_vector_sine"] = max((topk_sine(basis[:, [i]], vs[:, [j]]) for j, i in enumerate(idx)),
                                         default=0.0)
            out["vectors_checked"] = int(len(idx))
    return out


def parity_ok(p: dict, etol=1e-10, vtol=1e-8) -> bool:
    return (p["eig_rel_err"] <= etol and p["K"] == p["K_ref"] and p["topK_sine"] <= vtol
            and p.get("per_vector_sine", 0.0) <= vtol and p.get("cluster_sine", 0.0) <= vtol)
