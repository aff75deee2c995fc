"""Seeded synthetic inputs of BASELINE.json's configs — one
generator shared by bench.py, the tests and the golden-fixture scripts.

    A = X M + sigma N          (m x n, column-major, NOT centred: fit_pca centres)

X is a quantised Gaussian stream, M = R_X^-1 diag(s) V0^T on a fixed-point grid
(R_X = chol(X^T X), so X R_X^-1 = U0 has orthonormal columns; V0 the
CholeskyQR2 factor of a quantised Gaussian), N a Gaussian stream. Every
Gaussian is a pure function of (seed, stream, global element index)
(csrc/synth.h), X^T X and X M are exact in fp64 in any summation order, so:

* ``device_matrix`` (GPU, HBM) and ``host_matrix`` (CPU, numpy) return the same
  bytes for the same rows;
* a rank's row shard is byte-identical to those rows of the unsharded matrix
  (the per-rank partial X^T X are integers on a grid: their allreduce is exact).

Input synthesis only: nothing here is on the PCA path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

STREAM_X, STREAM_V, STREAM_NOISE = 1, 2, 3
MATRIX_SEED = 42      # the seed of A (bench.hpp:20's BenchConfig default)
METHOD_SEED = 4242    # Omega / Lanczos v0 seed of the sketch methods

SPECTRA = {
    "c1": lambda i: math.exp(-i / 20.0),
    "c2": lambda i: i ** -1.5,
    "c3": lambda i: math.exp(-i / 200.0),
    "c4": lambda i: 1.0 / i,
    "c5": lambda i: 1.0 / (1.0 + 0.01 * i),
}


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    sigma: float
    t: float
    method: str
    l: int = 0
    q: int = 0
    desc: str = ""

    def spectrum(self, n: int | None = None) -> np.ndarray:
        f = SPECTRA[self.name]
        return np.array([f(i) for i in range(1, (n or self.n) + 1)], dtype=np.float64)


# BASELINE.json configs[0..4]
CONFIGS = {
    "c1": Config("c1", 20000, 256, 1e-3, 0.95, "truncated",
                 desc="c1: truncated SVD via Gram, 20000x256, t=0.95"),
    "c2": Config("c2", 200000, 1024, 1e-3, 0.99, "randomized", l=1024, q=2,
                 desc="c2: randomized PCA 200000x1024, l=min(1024+10,1024), q=2, CholeskyQR2, t=0.99"),
    "c3": Config("c3", 500000, 2048, 1e-4, 0.95, "lanczos",
                 desc="c3: Lanczos on A^T A, 500000x2048, n steps, full reorth, t=0.95"),
    "c4": Config("c4", 8388608, 1024, 1e-3, 0.95, "truncated",
                 desc="c4: row-sharded truncated SVD 8388608x1024 (64 GB), t=0.95"),
    "c5": Config("c5", 65536, 4096, 1e-2, 0.90, "truncated",
                 desc="c5: full-spectrum truncated SVD 65536x4096, t=0.90"),
}


def _check(code: int) -> None:
    _lib.check(code)


def _vp(a) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr())


# --------------------------------------------------------------------------- host (CPU)
def host_block(seed: int, stream: int, m_total: int, row0: int, rows: int, cols: int,
               quantise: bool = False) -> np.ndarray:
    """Rows [row0, row0+rows) x cols of a Gaussian stream, Fortran order."""
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    _check(_lib.load().svdk_synth_fill(seed, stream, 1 if quantise else 0, m_total, row0, rows, cols,
                                       _vp(out), max(rows, 1)))
    return out


def host_add_noise(a: np.ndarray, seed: int, m_total: int, row0: int, sigma: float) -> np.ndarray:
    """a += sigma * N (rows [row0, row0 + a.shape[0]) of the noise stream), in place."""
    assert a.flags.f_contiguous and a.dtype == np.float64
    rows, cols = a.shape
    _check(_lib.load().svdk_synth_add_noise(seed, m_total, row0, rows, cols, float(sigma), _vp(a),
                                            max(rows, 1)))
    return a


def mixing(gx: np.ndarray, s: np.ndarray, seed: int) -> tuple[np.ndarray, float]:
    """M = R_X^-1 diag(s) V0^T on its fixed-point grid (host, deterministic)."""
    n = gx.shape[0]
    gx = np.asfortranarray(gx, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.float64)
    m = np.empty((n, n), dtype=np.float64, order="F")
    grid = C.c_double(0.0)
    _check(_lib.load().svdk_synth_mixing(n, _vp(gx), n, _vp(s), seed, _vp(m), n, C.byref(grid)))
    return m, grid.value


def host_gram_x(m_total: int, n: int, seed: int, chunk: int = 1 << 16) -> np.ndarray:
    """X^T X over all m_total rows (exact; numpy in any order)."""
    g = np.zeros((n, n))
    for r0 in range(0, m_total, chunk):
        x = host_block(seed, STREAM_X, m_total, r0, min(chunk, m_total - r0), n, quantise=True)
        g += x.T @ x
    return g


def host_matrix(m_total: int, n: int, s: np.ndarray, sigma: float, seed: int = MATRIX_SEED,
                row0: int = 0, rows: int | None = None, mix: np.ndarray | None = None) -> np.ndarray:
    """Rows [row0, row0+rows) of A = X M + sigma N on the CPU (Fortran order)."""
    rows = m_total - row0 if rows is None else rows
    if mix is None:
        mix, _ = mixing(host_gram_x(m_total, n, seed), s, seed)
    x = host_block(seed, STREAM_X, m_total, row0, rows, n, quantise=True)
    a = np.asfortranarray(x @ mix)
    del x
    if sigma:
        host_add_noise(a, seed, m_total, row0, sigma)
    return a


def config_host_matrix(cfg: Config | str, seed: int = MATRIX_SEED, row0: int = 0,
                       rows: int | None = None, mix=None) -> np.ndarray:
    cfg = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    return host_matrix(cfg.m, cfg.n, cfg.spectrum(), cfg.sigma, seed, row0, rows, mix)


# --------------------------------------------------------------------------- device (HBM)
def device_gram_x(eng, m_total: int, n: int, seed: int = MATRIX_SEED, row0: int = 0,
                  rows: int | None = None, chunk: int = 1 << 20):
    """X^T X over rows [row0, row0+rows) of the quantised stream, in HBM
    (svdk_dev_synth_fill + the engine's DMMA SYRK; exact). Everything runs on
    the engine's stream; the result is complete when this returns."""
    import torch

    from .engine import colmajor
    lib = _lib.load()
    rows = m_total - row0 if rows is None else rows
    dev = torch.device("cuda", eng.device)
    chunk = max(2, min(chunk, max(rows, 2)) & ~1)
    with torch.cuda.stream(eng.stream):
        x = colmajor(chunk, n, dev)
        g = torch.zeros(n, n, dtype=torch.float64, device=dev)
        gpart = torch.empty(n, n, dtype=torch.float64, device=dev)
        for r0 in range(0, rows, chunk):
            r = min(chunk, rows - r0)
            _check(lib.svdk_dev_synth_fill(eng.ctx.handle, seed, STREAM_X, 1, m_total, row0 + r0, r, n,
                                           _vp(x), x.stride(1)))
            eng.gram(x[:r], gpart.t())
            g += gpart
        del x, gpart
    eng.stream.synchronize()
    return g


def device_rows(eng, mix: np.ndarray, m_total: int, n: int, sigma: float, seed: int = MATRIX_SEED,
                row0: int = 0, rows: int | None = None, out=None, chunk: int = 1 << 20):
    """Rows [row0, row0+rows) of A = X M + sigma N in HBM, given the mixing
    matrix (engine stream; complete when this returns)."""
    import torch

    from .engine import colmajor
    lib = _lib.load()
    rows = m_total - row0 if rows is None else rows
    dev = torch.device("cuda", eng.device)
    chunk = max(2, min(chunk, max(rows, 2)) & ~1)
    with torch.cuda.stream(eng.stream):
        x = colmajor(chunk, n, dev)
        mdev = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(mix).T)).to(dev).t()  # column-major
        a = colmajor(rows, n, dev) if out is None else out
        for r0 in range(0, rows, chunk):
            r = min(chunk, rows - r0)
            _check(lib.svdk_dev_synth_fill(eng.ctx.handle, seed, STREAM_X, 1, m_total, row0 + r0, r, n,
                                           _vp(x), x.stride(1)))
            eng.gemm(x[:r], mdev, c=a[r0:r0 + r])
        if sigma and rows:
            _check(lib.svdk_dev_synth_add_noise(eng.ctx.handle, seed, m_total, row0, rows, n, float(sigma),
                                                _vp(a), a.stride(1)))
        del x, mdev
    eng.stream.synchronize()
    return a


def device_matrix(eng, m_total: int, n: int, s: np.ndarray, sigma: float, seed: int = MATRIX_SEED,
                  row0: int = 0, rows: int | None = None, allreduce=None, out=None,
                  chunk: int = 1 << 20):
    """Rows [row0, row0+rows) of A = X M + sigma N generated in HBM through
    the engine (quantised X by svdk_dev_synth_fill, X^T X by its DMMA SYRK, A
    = X M by its DMMA GEMM — all exact — then the noise). Multi-rank: pass
    the rank's row range and ``allreduce(tensor)`` summing the n x n partial
    Gram over ranks (exact on the grid). Returns a column-major tensor."""
    import torch
    g = device_gram_x(eng, m_total, n, seed, row0, rows, chunk)
    if allreduce is not None:
        allreduce(g)
        torch.cuda.synchronize(g.device)
    mix, _ = mixing(g.cpu().numpy(), s, seed)
    del g
    return device_rows(eng, mix, m_total, n, sigma, seed, row0, rows, out, chunk)


def config_device_matrix(eng, cfg: Config | str, seed: int = MATRIX_SEED, row0: int = 0,
                         rows: int | None = None, allreduce=None, out=None):
    cfg = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    return device_matrix(eng, cfg.m, cfg.n, cfg.spectrum(), cfg.sigma, seed, row0, rows, allreduce, out)
