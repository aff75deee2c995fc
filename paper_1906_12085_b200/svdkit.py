"""Host-side mirror of the reference svdkit API over the B200 engine's C-ABI.

Same names, argument meaning and error behaviour as the reference headers
(proj/include/svdkit/kernels.hpp, svd_methods.hpp, pca.hpp); matrices are
numpy float64 arrays (converted to column-major, the reference DenseMatrix
layout, dense_matrix.hpp:41-46). Every compute call goes through
libsvdk.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .errors import DimensionError, ParamError

__all__ = [
    "RngSeed", "SvdMethod", "Orientation", "MethodParams", "QrResult", "EigResult", "SvdResult",
    "CenterResult", "PcaModel", "matmul", "matmul_transposed_left", "transpose", "gram",
    "frobenius_norm_sq", "frobenius_norm", "qr_thin", "eig_sym", "gaussian_matrix",
    "truncated_svd", "randomized_pca", "krylov_svd", "lanczos_svd", "compute_svd",
    "compute_svd_any", "method_name", "method_from_name", "center", "total_variance",
    "select_components", "fit_pca", "transform", "residual_delta", "truncate_rank",
]


# ---------------------------------------------------------------- value types
@dataclass(frozen=True)
class RngSeed:
    """kernels.hpp:14-16"""
    value: int = 0


class SvdMethod(enum.IntEnum):
    """svd_methods.hpp:13 (+ Lanczos, new in this engine)."""
    Truncated = 0
    Randomized = 1
    Krylov = 2
    Lanczos = 3


class Orientation(enum.IntEnum):
    """pca.hpp:16"""
    ColumnsAreExamples = 0
    RowsAreExamples = 1


@dataclass
class MethodParams:
    """svd_methods.hpp:20-27; sketch_width = l, power_iterations = q / Krylov depth
    (for Lanczos: sketch_width = number of steps, 0 = n)."""
    sketch_width: int = 1
    power_iterations: int = 1
    seed: RngSeed = field(default_factory=RngSeed)

    @staticmethod
    def defaults_for(n: int, seed: RngSeed = RngSeed(0)) -> "MethodParams":
        """svd_methods.cpp:30-32: l = ceil(n/2), one power iteration."""
        return MethodParams((n + 1) // 2, 1, seed)


@dataclass
class QrResult:
    q: np.ndarray
    r: np.ndarray
    rank: int


@dataclass
class EigResult:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray


@dataclass
class SvdResult:
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray
    rank: int = 0
    method: SvdMethod = SvdMethod.Truncated


@dataclass
class CenterResult:
    centered: np.ndarray
    mean: np.ndarray


@dataclass
class PcaModel:
    basis: np.ndarray
    eigenvalues: np.ndarray
    total_variance: float
    orientation: Orientation
    mean: np.ndarray


_NAMES = {SvdMethod.Truncated: "truncated", SvdMethod.Randomized: "randomized",
          SvdMethod.Krylov: "krylov", SvdMethod.Lanczos: "lanczos"}


def method_name(method: SvdMethod) -> str:
    """svd_methods.cpp:11-21"""
    return _NAMES.get(SvdMethod(method), "unknown")


def method_from_name(name: str) -> Optional[SvdMethod]:
    """svd_methods.cpp:23-28"""
    for k, v in _NAMES.items():
        if v == name:
            return k
    return None


# ---------------------------------------------------------------- helpers
def _mat(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise DimensionError(f"expected a matrix, got shape {a.shape}")
    return np.asfortranarray(a)


def _finite(a: np.ndarray) -> np.ndarray:
    # DenseMatrix rejects NaN/Inf on construction (dense_matrix.cpp:13-19)
    if not np.isfinite(a).all():
        raise ParamError("DenseMatrix: non-finite entry (NaN/Inf) rejected")
    return a


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _shape(a: np.ndarray) -> str:
    return f"{a.shape[0]}x{a.shape[1]}"


def _ctx():
    return _lib.default_context().handle


def _out(rows: int, cols: int) -> np.ndarray:
    return np.zeros((rows, cols), dtype=np.float64, order="F")


# ---------------------------------------------------------------- L1 kernels
def matmul(a, b) -> np.ndarray:
    """kernels.cpp:14-45 — C = A B; NumericalError on a non-finite result."""
    a, b = _mat(a), _mat(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionError(f"matmul: inner dimensions differ, a is {_shape(a)}, b is {_shape(b)}")
    c = _out(a.shape[0], b.shape[1])
    _lib.check(_lib.load().svdk_matmul(_ctx(), _ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[1], _ptr(c)))
    return c


def matmul_transposed_left(a, b) -> np.ndarray:
    """kernels.cpp:47-67 — C = A^T B without forming A^T."""
    a, b = _mat(a), _mat(b)
    if a.shape[0] != b.shape[0]:
        raise DimensionError(
            f"matmul_transposed_left: row counts differ, a is {_shape(a)}, b is {_shape(b)}")
    c = _out(a.shape[1], b.shape[1])
    _lib.check(_lib.load().svdk_matmul_transposed_left(_ctx(), _ptr(a), a.shape[0], a.shape[1], _ptr(b),
                                                       b.shape[1], _ptr(c)))
    return c


def transpose(a) -> np.ndarray:
    """kernels.cpp:69-78"""
    a = _mat(a)
    t = _out(a.shape[1], a.shape[0])
    _lib.check(_lib.load().svdk_transpose(_ctx(), _ptr(a), a.shape[0], a.shape[1], _ptr(t)))
    return t


def gram(a) -> np.ndarray:
    """kernels.cpp:80-97 — exactly symmetric A^T A."""
    a = _mat(a)
    n = a.shape[1]
    g = _out(n, n)
    _lib.check(_lib.load().svdk_gram(_ctx(), _ptr(a), a.shape[0], n, _ptr(g)))
    return g


def frobenius_norm_sq(a) -> float:
    """kernels.cpp:99-105"""
    a = _mat(a)
    out = C.c_double(0.0)
    _lib.check(_lib.load().svdk_frobenius_norm_sq(_ctx(), _ptr(a), a.shape[0], a.shape[1], C.byref(out)))
    return out.value


def frobenius_norm(a) -> float:
    """kernels.cpp:107-109"""
    return float(np.sqrt(frobenius_norm_sq(a)))


def qr_thin(h) -> QrResult:
    """kernels.cpp:111-224 — thin QR (CholeskyQR2 on the engine), R with
    nonnegative diagonal; DimensionError when rows < cols."""
    h = _mat(h)
    m, p = h.shape
    if m < p:
        raise DimensionError(f"qr_thin: need rows >= cols, got {_shape(h)}")
    q, r = _out(m, p), _out(p, p)
    rank = C.c_int64(0)
    _lib.check(_lib.load().svdk_qr_thin(_ctx(), _ptr(h), m, p, _ptr(q), _ptr(r), C.byref(rank)))
    return QrResult(q, r, int(rank.value))


def eig_sym(s, max_sweeps: int = 30) -> EigResult:
    """kernels.cpp:241-346 — Jacobi eigendecomposition, descending stable order."""
    s = _mat(s)
    n = s.shape[0]
    if s.shape[0] != s.shape[1]:
        raise DimensionError(f"eig_sym: matrix not square, got {_shape(s)}")
    w = np.zeros(n)
    v = _out(n, n)
    _lib.check(_lib.load().svdk_eig_sym(_ctx(), _ptr(s), n, int(max_sweeps), _ptr(w), _ptr(v)))
    return EigResult(w, v)


def gaussian_matrix(rows: int, cols: int, seed=RngSeed(0)) -> np.ndarray:
    """kernels.cpp:348-379 — bit-identical mt19937_64 + Box-Muller sample."""
    seed = seed.value if isinstance(seed, RngSeed) else int(seed)
    if rows < 1 or cols < 1:
        raise ParamError("gaussian_matrix: rows and cols must be >= 1")
    g = _out(rows, cols)
    _lib.check(_lib.load().svdk_gaussian_matrix(rows, cols, seed & (2**64 - 1), _ptr(g)))
    return g


# ---------------------------------------------------------------- L2 methods
def _svd_call(fn, a: np.ndarray, width: int, *extra, method=SvdMethod.Truncated) -> SvdResult:
    m, n = a.shape
    u, v = _out(m, max(width, 1)), _out(n, max(width, 1))
    s = np.zeros(max(width, n, 1))
    rank = C.c_int64(0)
    _lib.check(fn(_ctx(), _ptr(a), m, n, *extra, _ptr(u), _ptr(s), _ptr(v), C.byref(rank)))
    r = int(rank.value)
    return SvdResult(np.asfortranarray(u[:, :r]), s[:r].copy(), np.asfortranarray(v[:, :r]), r, method)


def truncated_svd(a) -> SvdResult:
    """svd_methods.cpp:121-158 — Gram route: eig(A^T A), sigma = sqrt, U = A V / sigma."""
    a = _finite(_mat(a))
    return _svd_call(_lib.load().svdk_truncated_svd, a, a.shape[1], method=SvdMethod.Truncated)


def randomized_pca(a, p: MethodParams) -> SvdResult:
    """svd_methods.cpp:160-170"""
    a = _finite(_mat(a))
    return _svd_call(_lib.load().svdk_randomized_pca, a, max(int(p.sketch_width), 1), int(p.sketch_width),
                     int(p.power_iterations), p.seed.value & (2**64 - 1), method=SvdMethod.Randomized)


def krylov_svd(a, p: MethodParams) -> SvdResult:
    """svd_methods.cpp:172-196 — block Krylov [A G | A(A^T A G) | ...]."""
    a = _finite(_mat(a))
    w = min(max(int(p.power_iterations) + 1, 1) * max(int(p.sketch_width), 1), a.shape[1])
    return _svd_call(_lib.load().svdk_krylov_svd, a, w, int(p.sketch_width), int(p.power_iterations),
                     p.seed.value & (2**64 - 1), method=SvdMethod.Krylov)


def lanczos_svd(a, steps: int = 0, seed=RngSeed(0)) -> SvdResult:
    """NEW (no reference): Lanczos on A^T A with full reorthogonalisation."""
    a = _finite(_mat(a))
    seed = seed.value if isinstance(seed, RngSeed) else int(seed)
    n = a.shape[1]
    w = n if steps <= 0 or steps > n else steps
    return _svd_call(_lib.load().svdk_lanczos_svd, a, w, int(steps), seed & (2**64 - 1),
                     method=SvdMethod.Lanczos)


def compute_svd(a, method: SvdMethod, p: MethodParams) -> SvdResult:
    """svd_methods.cpp:227-237"""
    method = SvdMethod(method)
    if method == SvdMethod.Truncated:
        return truncated_svd(a)
    if method == SvdMethod.Randomized:
        return randomized_pca(a, p)
    if method == SvdMethod.Krylov:
        return krylov_svd(a, p)
    return lanczos_svd(a, p.sketch_width, p.seed)


def compute_svd_any(a, method: SvdMethod, p: MethodParams) -> SvdResult:
    """svd_methods.cpp:239-246 — wide input: factor A^T and swap U/V."""
    a = _mat(a)
    if a.shape[0] >= a.shape[1]:
        return compute_svd(a, method, p)
    s = compute_svd(np.asfortranarray(a.T), method, p)
    s.u, s.v = s.v, s.u
    return s


# ---------------------------------------------------------------- L3 PCA
def center(a, orientation: Orientation) -> CenterResult:
    """pca.cpp:13-55"""
    a = _mat(a)
    m, n = a.shape
    nm = m if Orientation(orientation) == Orientation.ColumnsAreExamples else n
    c, mean = _out(m, n), np.zeros(max(nm, 1))
    _lib.check(_lib.load().svdk_center(_ctx(), _ptr(a), m, n, int(orientation), _ptr(c), _ptr(mean)))
    return CenterResult(c, mean[:nm].copy())


def total_variance(centered) -> float:
    """pca.cpp:57-59 — ||A||_F^2."""
    return frobenius_norm_sq(centered)


def select_components(eigenvalues, total: float, threshold: float) -> Optional[int]:
    """pca.cpp:61-89 — smallest K >= 1 reaching the explained-variance
    threshold, None when the stored spectrum falls short."""
    w = np.ascontiguousarray(np.asarray(eigenvalues, dtype=np.float64))
    k = C.c_int64(0)
    _lib.check(_lib.load().svdk_select_components(_ctx(), _ptr(w) if w.size else None, w.size,
                                                  float(total), float(threshold), C.byref(k)))
    return int(k.value) if k.value > 0 else None


def fit_pca(data, orientation: Orientation, method: SvdMethod, params: MethodParams,
            center_data: bool = True) -> PcaModel:
    """pca.cpp:91-116"""
    a = _finite(_mat(data))
    m, n = a.shape
    orientation = Orientation(orientation)
    nm = m if orientation == Orientation.ColumnsAreExamples else n
    tall_n = min(m, n)
    basis_rows = m if orientation == Orientation.ColumnsAreExamples else n
    method = SvdMethod(method)
    if method == SvdMethod.Randomized:
        width = int(params.sketch_width)
    elif method == SvdMethod.Krylov:
        width = min((int(params.power_iterations) + 1) * int(params.sketch_width), tall_n)
    elif method == SvdMethod.Lanczos:
        width = tall_n if params.sketch_width <= 0 or params.sketch_width > tall_n else int(params.sketch_width)
    else:
        width = tall_n
    width = max(width, 1)
    basis, eig = _out(basis_rows, width), np.zeros(width)
    mean = np.zeros(max(nm, 1))
    total = C.c_double(0.0)
    rank = C.c_int64(0)
    _lib.check(_lib.load().svdk_fit_pca(_ctx(), _ptr(a), m, n, int(orientation), int(method),
                                        int(params.sketch_width), int(params.power_iterations),
                                        params.seed.value & (2**64 - 1), 1 if center_data else 0,
                                        _ptr(basis), _ptr(eig), C.byref(total), _ptr(mean), C.byref(rank)))
    r = int(rank.value)
    return PcaModel(np.asfortranarray(basis[:, :r]), eig[:r].copy(), total.value, orientation, mean[:nm].copy())


def transform(model: PcaModel, a) -> np.ndarray:
    """pca.cpp:118-131 — project centred data onto the basis."""
    a = _mat(a)
    if model.orientation == Orientation.ColumnsAreExamples:
        if a.shape[0] != model.basis.shape[0]:
            raise DimensionError(f"transform: data is {_shape(a)} but basis is {_shape(model.basis)} "
                                 "(feature rows must match)")
        return matmul_transposed_left(model.basis, a)
    if a.shape[1] != model.basis.shape[0]:
        raise DimensionError(f"transform: data is {_shape(a)} but basis is {_shape(model.basis)} "
                             "(feature columns must match)")
    return matmul(a, model.basis)


def residual_delta(a, s: SvdResult) -> float:
    """pca.cpp:133-168 — ||A - U diag(sigma) V^T||_F / ||A||_F on the GPU."""
    a = _mat(a)
    u, v = _mat(s.u), _mat(s.v)
    if u.shape[0] != a.shape[0] or v.shape[0] != a.shape[1]:
        raise DimensionError(f"residual_delta: factors {_shape(u)}/{_shape(v)} do not match data {_shape(a)}")
    sig = np.ascontiguousarray(s.sigma, dtype=np.float64)
    out = C.c_double(0.0)
    _lib.check(_lib.load().svdk_residual_delta(_ctx(), _ptr(a), a.shape[0], a.shape[1], _ptr(u), _ptr(sig),
                                               _ptr(v), int(s.rank), C.byref(out)))
    return out.value


def truncate_rank(s: SvdResult, k: int) -> SvdResult:
    """svd_methods.cpp:198-225 — keep the leading k triplets (pure data movement)."""
    if k < 1 or k > s.rank:
        raise ParamError(f"truncate_rank: k = {k} outside [1, rank = {s.rank}]")
    return SvdResult(np.asfortranarray(s.u[:, :k]), s.sigma[:k].copy(), np.asfortranarray(s.v[:, :k]), k, s.method)
