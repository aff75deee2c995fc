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
