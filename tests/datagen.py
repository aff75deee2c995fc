"""Deterministic synthetic inputs (BASELINE.json configs) — test infrastructure.

Every matrix comes from the ONE generator shared with bench.py and the
fixture scripts (paper_1906_12085_b200/synth.py, csrc/synth.h):
A = X M + noise * N with X, N counter-based Gaussian streams keyed by the
global element index and M = R_X^-1 diag(s) V0^T on a fixed-point grid, so
the same bytes come out on this container's CPU, on the GPU box's CPU and in
HBM (``synth.device_matrix``).

``make_matrix`` returns the column-centred matrix (centring by the C oracle's
restatement of the reference's ``center``, fixed loop order) for the small
generic cases; ``config_matrix`` returns a BASELINE config's raw A, which the
pipeline under test centres itself (fit_pca with center = true), exactly as
the golden fixtures' reference runs did.
"""
from __future__ import annotations

import numpy as np

from paper_1906_12085_b200 import synth

SPECTRA = synth.SPECTRA
NOISE = {k: c.sigma for k, c in synth.CONFIGS.items()}
SHAPES = {k: (c.m, c.n) for k, c in synth.CONFIGS.items()}
THRESHOLD = {k: c.t for k, c in synth.CONFIGS.items()}

_CACHE = {}


def spectrum(spec, n: int) -> np.ndarray:
    f = SPECTRA[spec] if isinstance(spec, str) else spec
    return np.array([f(i) for i in range(1, n + 1)], dtype=np.float64)


def make_matrix(m: int, n: int, spectrum_name="c1", noise=None, seed: int = 42, center: bool = True,
                oracle=None) -> np.ndarray:
    key = (m, n, spectrum_name if isinstance(spectrum_name, str) else id(spectrum_name), noise, seed, center)
    if key not in _CACHE:
        _CACHE[key] = _make(m, n, spectrum_name, noise, seed, center, oracle)
        _CACHE[key].setflags(write=False)
    return _CACHE[key]


def _make(m, n, spec, noise, seed, center, oracle):
    if noise is None:
        noise = NOISE[spec] if isinstance(spec, str) else 0.0
    a = synth.host_matrix(m, n, spectrum(spec, n), noise, seed)
    if center:
        from oracle.pyoracle import Oracle
        orc = oracle or Oracle("port")
        a = orc.center(a, 1)[0]
    return np.asfortranarray(a)


def config_matrix(name: str, seed: int = synth.MATRIX_SEED, rows: int | None = None) -> np.ndarray:
    """BASELINE config `name`'s raw (uncentred) A, or its first `rows` rows."""
    cfg = synth.CONFIGS[name]
    key = ("cfg", name, seed, rows)
    if key not in _CACHE:
        a = synth.config_host_matrix(cfg, seed, 0, rows)
        a.setflags(write=False)
        _CACHE[key] = a
    return _CACHE[key]
