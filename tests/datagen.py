"""Deterministic synthetic inputs (BASELINE.json configs) — test infrastructure.

A = U0 diag(s) V0^T + noise * N, column-centred, with U0 / V0 the Q factors
of seeded Gaussians. Randomness comes from numpy's PCG64 (platform
independent); every floating-point reduction goes through the C oracle
(fixed loop order, -ffp-contract=off), so the same bytes come out on this
container and on the GPU box.
"""
from __future__ import annotations

import numpy as np

SPECTRA = {
    "c1": lambda i: np.exp(-i / 20.0),
    "c2": lambda i: i ** -1.5,
    "c3": lambda i: np.exp(-i / 200.0),
    "c4": lambda i: 1.0 / i,
    "c5": lambda i: 1.0 / (1.0 + 0.01 * i),
}
NOISE = {"c1": 1e-3, "c2": 1e-3, "c3": 1e-4, "c4": 1e-3, "c5": 1e-2}
SHAPES = {"c1": (20000, 256), "c2": (200000, 1024), "c3": (500000, 2048), "c4": (8388608, 1024),
          "c5": (65536, 4096)}
THRESHOLD = {"c1": 0.95, "c2": 0.99, "c3": 0.95, "c4": 0.95, "c5": 0.90}


_CACHE = {}


def make_matrix(m: int, n: int, spectrum="c1", noise=None, seed: int = 42, center: bool = True,
                oracle=None) -> np.ndarray:
    key = (m, n, spectrum if isinstance(spectrum, str) else id(spectrum), noise, seed, center)
    if key not in _CACHE:
        _CACHE[key] = _make(m, n, spectrum, noise, seed, center, oracle)
        _CACHE[key].setflags(write=False)
    return _CACHE[key]


def _make(m, n, spectrum, noise, seed, center, oracle):
    from oracle.pyoracle import Oracle
    orc = oracle or Oracle("port")
    f = SPECTRA[spectrum] if isinstance(spectrum, str) else spectrum
    noise = NOISE[spectrum] if (noise is None and isinstance(spectrum, str)) else (noise or 0.0)
    rng = np.random.default_rng(seed)
    g1 = np.asfortranarray(rng.standard_normal((n, m)).T)
    u0 = orc.qr_thin(g1)[0]
    g2 = np.asfortranarray(rng.standard_normal((n, n)).T)
    v0 = orc.qr_thin(g2)[0]
    s = f(np.arange(1, n + 1, dtype=np.float64))
    a = orc.matmul(np.asfortranarray(u0 * s), np.asfortranarray(v0.T))
    if noise:
        a = a + noise * np.asfortranarray(rng.standard_normal((n, m)).T)
    a = np.asfortranarray(a)
    if center:
        a = orc.center(a, 1)[0]
    return a
