"""Device-resident entry points (svdk_dev_* in include/svdk.h) over torch CUDA tensors.

Matrices are column-major torch float64 tensors of shape (rows, cols) with
stride (1, ld) — create them as ``torch.empty(cols, ld, ...).t()[:rows]`` or
with :func:`colmajor`. torch is only the allocator/stream owner here; all
compute is libsvdk.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib
from .errors import DimensionError

try:
    import torch
except ImportError:  # pragma: no cover - torch is in the image
    torch = None


def colmajor(rows: int, cols: int, device="cuda", ld: int | None = None):
    """Uninitialised column-major (rows x cols) float64 tensor with an even leading dimension."""
    ld = ld or max(2, rows + (rows & 1))
    return torch.empty(cols, ld, dtype=torch.float64, device=device).t()[:rows]


def _ld(t) -> int:
    if t.dim() != 2 or t.dtype != torch.float64 or not t.is_cuda:
        raise DimensionError("expected a 2-D float64 CUDA tensor")
    if t.shape[1] > 1 and t.stride(0) != 1:
        raise DimensionError("expected a column-major tensor (stride(0) == 1)")
    return max(int(t.stride(1)), int(t.shape[0]), 1)


def _p(t):
    return C.c_void_p(t.data_ptr())


@dataclass
class PcaOutput:
    u: "torch.Tensor"
    sigma: "torch.Tensor"
    v: "torch.Tensor"
    mean: "torch.Tensor"
    rank: int
    k: int | None
    total: float


class Engine:
    """One svdk context bound to torch's current CUDA stream on `device`."""

    def __init__(self, device: int = 0, stream=None):
        self.ctx = _lib.Context(device)
        self.device = device
        # A dedicated (non-default) torch stream: the engine captures CUDA
        # graphs on it, which the legacy default stream does not allow.
        self.stream = stream if stream is not None else torch.cuda.Stream(device)
        self.ctx.set_stream(self.stream.cuda_stream)

    @property
    def lib(self):
        return _lib.load()

    def launches(self) -> int:
        return self.ctx.launches()

    def gram(self, a, g=None):
        m, n = a.shape
        g = colmajor(n, n, a.device, ld=n) if g is None else g
        _lib.check(self.lib.svdk_dev_gram(self.ctx.handle, _p(a), m, n, _ld(a), _p(g), _ld(g)))
        return g

    def gemm(self, a, b, transa: bool = False, c=None):
        if transa:
            k, m = a.shape
        else:
            m, k = a.shape
        if b.shape[0] != k:
            raise DimensionError("gemm: inner dimensions differ")
        n = b.shape[1]
        c = colmajor(m, n, a.device) if c is None else c
        _lib.check(self.lib.svdk_dev_gemm(self.ctx.handle, 1 if transa else 0, m, n, k, _p(a), _ld(a),
                                          _p(b), _ld(b), _p(c), _ld(c)))
        return c

    def gemv_pair(self, a, q, w=None):
        """w = A^T (A q) (the Lanczos matvec pair)."""
        m, n = a.shape
        w = torch.empty(n, dtype=torch.float64, device=a.device) if w is None else w
        _lib.check(self.lib.svdk_dev_gemv_pair(self.ctx.handle, _p(a), m, n, _ld(a), _p(q), _p(w)))
        return w

    def eig_sym(self, s, max_sweeps: int = 30):
        n = s.shape[0]
        w = torch.empty(n, dtype=torch.float64, device=s.device)
        v = colmajor(n, n, s.device, ld=n)
        _lib.check(self.lib.svdk_dev_eig_sym(self.ctx.handle, _p(s), n, _ld(s), int(max_sweeps), _p(w), _p(v), n))
        return w, v

    def qr_thin(self, h):
        m, p = h.shape
        q = colmajor(m, p, h.device)
        r = colmajor(p, p, h.device, ld=p)
        rank = C.c_int64(0)
        _lib.check(self.lib.svdk_dev_qr_thin(self.ctx.handle, _p(h), m, p, _ld(h), _p(q), _ld(q), _p(r),
                                             C.byref(rank)))
        return q, r, int(rank.value)

    def pca(self, a, method: int = 0, l: int = 0, q: int = 0, seed: int = 0, center=True,
            threshold: float = 0.95, out: PcaOutput | None = None) -> PcaOutput:
        """Full RowsAreExamples PCA on a device-resident (row shard of) A.
        center: True/1 centre a copy, 2 centre A in place (overwrites A), False/0 none.
        The call returns after the engine's stream has produced K (the outputs
        are complete); the other entry points are asynchronous on ``self.stream``."""
        m, n = a.shape
        width = {1: l, 2: min((q + 1) * l, n), 3: (n if l <= 0 or l > n else l)}.get(int(method), n)
        width = max(width, 1)
        if out is None:
            with torch.cuda.stream(self.stream):  # outputs belong to the engine's stream
                out = PcaOutput(colmajor(m, width, a.device),
                                torch.empty(max(width, n), dtype=torch.float64, device=a.device),
                                colmajor(n, width, a.device, ld=n), torch.empty(n, dtype=torch.float64, device=a.device),
                                0, None, 0.0)
        rank, k, total = C.c_int64(0), C.c_int64(0), C.c_double(0.0)
        _lib.check(self.lib.svdk_dev_pca(self.ctx.handle, _p(a), m, n, _ld(a), int(method), int(l), int(q),
                                         int(seed) & (2**64 - 1), int(center), float(threshold),
                                         _p(out.u), _ld(out.u), _p(out.sigma), _p(out.v), n, _p(out.mean),
                                         C.byref(rank), C.byref(k), C.byref(total)))
        out.rank, out.k, out.total = int(rank.value), (int(k.value) or None), total.value
        return out
