"""ctypes wrappers for the parity CHECKERS — test infrastructure only.

Two interchangeable backends with the same Python surface:
  Oracle("port") -> oracle/liboracle.so        (C restatement, svdk_oracle.c)
  Oracle("ref")  -> oracle/_ref/libsvdkit_ref.so (the unmodified reference
                     sources compiled in place + ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libsvdkit_ref.so")

_sz = C.c_size_t
_vp = C.c_void_p


class OracleError(RuntimeError):
    def __init__(self, code: int, residual: float = 0.0):
        super().__init__({1: "DimensionError", 2: "ParamError", 3: "NumericalError"}.get(code, f"error {code}"))
        self.code = code
        self.residual = residual


def build(quiet: bool = True) -> None:
    """Build liboracle.so (+ _ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def available(kind: str) -> bool:
    return os.path.exists(PORT_PATH if kind == "port" else REF_PATH)


@dataclass
class Svd:
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray
    rank: int


def _F(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return _vp(a.ctypes.data)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_PATH if kind == "port" else REF_PATH
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.pre = "orc_" if kind == "port" else "ref_"
        for fn in ("gram", "matmul", "matmul_tl", "qr_thin", "truncated_svd", "randomized_pca",
                   "krylov_svd", "center", "select_components", "gaussian_matrix", "eig_sym"):
            getattr(self.lib, self.pre + fn).restype = C.c_int
        getattr(self.lib, self.pre + "frobenius_norm_sq").restype = C.c_double

    def _f(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, code, residual=0.0):
        if code != 0:
            if self.kind == "ref" and code == 3:
                self.lib.ref_last_residual.restype = C.c_double
                residual = self.lib.ref_last_residual()
            raise OracleError(code, residual)

    # kernels.cpp
    def gaussian_matrix(self, rows, cols, seed):
        out = np.zeros((rows, cols), order="F")
        self._check(self._f("gaussian_matrix")(_sz(rows), _sz(cols), C.c_uint64(seed), _p(out)))
        return out

    def matmul(self, a, b):
        a, b = _F(a), _F(b)
        c = np.zeros((a.shape[0], b.shape[1]), order="F")
        self._check(self._f("matmul")(_p(a), _sz(a.shape[0]), _sz(a.shape[1]), _p(b), _sz(b.shape[1]), _p(c)))
        return c

    def matmul_tl(self, a, b):
        a, b = _F(a), _F(b)
        c = np.zeros((a.shape[1], b.shape[1]), order="F")
        self._check(self._f("matmul_tl")(_p(a), _sz(a.shape[0]), _sz(a.shape[1]), _p(b), _sz(b.shape[1]), _p(c)))
        return c

    def gram(self, a):
        a = _F(a)
        g = np.zeros((a.shape[1], a.shape[1]), order="F")
        self._check(self._f("gram")(_p(a), _sz(a.shape[0]), _sz(a.shape[1]), _p(g)))
        return g

    def frobenius_norm_sq(self, a):
        a = _F(a)
        if self.kind == "port":
            return self._f("frobenius_norm_sq")(_p(a), _sz(a.size))
        return self._f("frobenius_norm_sq")(_p(a), _sz(a.shape[0]), _sz(a.shape[1]))

    def qr_thin(self, h):
        h = _F(h)
        m, p = h.shape
        q, r = np.zeros((m, p), order="F"), np.zeros((p, p), order="F")
        rank = _sz(0)
        self._check(self._f("qr_thin")(_p(h), _sz(m), _sz(p), _p(q), _p(r), C.byref(rank)))
        return q, r, rank.value

    def eig_sym(self, s, max_sweeps=30):
        s = _F(s)
        n = s.shape[0]
        w, v = np.zeros(n), np.zeros((n, n), order="F")
        if self.kind == "port":
            res = C.c_double(0.0)
            sw = C.c_int(0)
            code = self._f("eig_sym")(_p(s), _sz(n), C.c_int(max_sweeps), _p(w), _p(v), C.byref(res), C.byref(sw))
            self._check(code, res.value)
        else:
            self._check(self._f("eig_sym")(_p(s), _sz(n), C.c_int(max_sweeps), _p(w), _p(v)))
        return w, v

    def _svd(self, fn, a, width, *extra):
        a = _F(a)
        m, n = a.shape
        width = max(width, 1)
        u, v = np.zeros((m, width), order="F"), np.zeros((n, width), order="F")
        s = np.zeros(max(width, n))
        rank = _sz(0)
        self._check(fn(_p(a), _sz(m), _sz(n), *extra, _p(u), _p(s), _p(v), C.byref(rank)))
        r = rank.value
        return Svd(np.asfortranarray(u[:, :r]), s[:r].copy(), np.asfortranarray(v[:, :r]), r)

    def truncated_svd(self, a):
        return self._svd(self._f("truncated_svd"), a, np.shape(a)[1])

    def randomized_pca(self, a, l, q, seed):
        return self._svd(self._f("randomized_pca"), a, l, _sz(l), _sz(q), C.c_uint64(seed))

    def krylov_svd(self, a, l, i, seed):
        w = min((i + 1) * l, np.shape(a)[1])
        return self._svd(self._f("krylov_svd"), a, w, _sz(l), _sz(i), C.c_uint64(seed))

    def center(self, a, orientation):
        a = _F(a)
        m, n = a.shape
        c = np.zeros((m, n), order="F")
        mean = np.zeros(m if orientation == 0 else n)
        self._check(self._f("center")(_p(a), _sz(m), _sz(n), C.c_int(orientation), _p(c), _p(mean)))
        return c, mean

    def select_components(self, w, total, threshold):
        w = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
        k = _sz(0)
        self._check(self._f("select_components")(_p(w) if w.size else None, _sz(w.size), C.c_double(total),
                                                  C.c_double(threshold), C.byref(k)))
        return k.value or None

    def fit_pca_rows(self, a, method="truncated", l=1, q=1, seed=0):
        """fit_pca(RowsAreExamples, method, center=True) -> (eigenvalues, basis V, total, mean)."""
        c, mean = self.center(a, 1)
        total = self.frobenius_norm_sq(c)
        if method == "truncated":
            s = self.truncated_svd(c)
        elif method == "randomized":
            s = self.randomized_pca(c, l, q, seed)
        else:
            s = self.krylov_svd(c, l, q, seed)
        return s.sigma ** 2, s.v, total, mean

    def residual_delta(self, a, u, sigma, v):
        """pca.cpp:133-168 (reference only)."""
        if self.kind != "ref":
            rec = (u * sigma) @ v.T
            return float(np.sqrt(((a - rec) ** 2).sum() / (a ** 2).sum()))
        a, u, v = _F(a), _F(u), _F(v)
        s = np.ascontiguousarray(sigma, dtype=np.float64)
        d = C.c_double(0.0)
        self.lib.ref_residual_delta.restype = C.c_int
        self._check(self.lib.ref_residual_delta(_p(a), _sz(a.shape[0]), _sz(a.shape[1]), _p(u), _p(s), _p(v),
                                                _sz(len(s)), C.byref(d)))
        return d.value


class RefTools:
    """The reference's host-side tools (cost model, CSV / IDX formats, bench grid
    text) through ref_shim.cpp — parity checker for the engine's versions."""

    def __init__(self):
        lib = C.CDLL(REF_PATH)
        self.lib = lib
        lib.ref_last_offset.restype = _sz
        lib.ref_sketch_width_for.restype = _sz
        lib.ref_sketch_width_for.argtypes = [C.c_double, _sz]
        lib.ref_format_double.argtypes = [C.c_double, C.c_char_p, _sz]

    def _status(self, code):
        if code != 0:
            err = OracleError(code)
            err.offset = int(self.lib.ref_last_offset()) if code == 8 else 0
            raise err

    def cost(self, model, m, n, l=0, i=0):
        f, e, b = C.c_double(), C.c_double(), C.c_double()
        self._status(self.lib.ref_cost_model(C.c_int(model), _sz(m), _sz(n), _sz(l), _sz(i),
                                             C.byref(f), C.byref(e), C.byref(b)))
        return f.value, e.value, b.value

    def format_double(self, v: float) -> str:
        buf = C.create_string_buffer(64)
        assert self.lib.ref_format_double(C.c_double(v), buf, 64) == 0
        return buf.value.decode()

    def idx_parse(self, data: bytes):
        dims = (C.c_uint64 * 3)()
        buf = C.create_string_buffer(data, len(data)) if data else None
        self._status(self.lib.ref_idx_parse(buf, _sz(len(data)), dims))
        return tuple(int(x) for x in dims)

    def images_to_matrix(self, data: bytes):
        c, h, w = self.idx_parse(data)
        out = np.zeros((c, h * w), order="F")
        buf = C.create_string_buffer(data, len(data))
        self._status(self.lib.ref_images_to_matrix(buf, _sz(len(data)), _p(out)))
        return out

    def image_as_matrix(self, data: bytes, index: int):
        c, h, w = self.idx_parse(data)
        out = np.zeros((h, w), order="F")
        buf = C.create_string_buffer(data, len(data))
        self._status(self.lib.ref_image_as_matrix(buf, _sz(len(data)), _sz(index), _p(out)))
        return out

    def sketch_width_for(self, l_fraction: float, n: int) -> int:
        return int(self.lib.ref_sketch_width_for(l_fraction, n))

    def expand_grid(self, rows, cols):
        r = (C.c_size_t * max(1, len(rows)))(*rows)
        c = (C.c_size_t * max(1, len(cols)))(*cols)
        out = (C.c_size_t * max(2, 2 * len(rows) * len(cols)))()
        cells = _sz(0)
        self._status(self.lib.ref_expand_grid(r, _sz(len(rows)), c, _sz(len(cols)), out, C.byref(cells)))
        return [(int(out[2 * k]), int(out[2 * k + 1])) for k in range(cells.value)]

    def _records(self, recs):
        k = len(recs)
        meth = (C.c_int * max(1, k))(*[int(r[0]) for r in recs])
        m = (C.c_size_t * max(1, k))(*[r[1] for r in recs])
        n = (C.c_size_t * max(1, k))(*[r[2] for r in recs])
        rep = (C.c_size_t * max(1, k))(*[r[3] for r in recs])
        cols = (C.c_double * max(1, 5 * k))(*[x for r in recs for x in r[4:9]])
        return meth, m, n, rep, cols, _sz(k)

    def bench_csv(self, recs) -> str:
        """recs: tuples (method, m, n, repeats, mean, std, delta, flops, bytes)."""
        buf = C.create_string_buffer(1 << 20)
        assert self.lib.ref_bench_csv(*self._records(recs), buf, _sz(1 << 20)) == 0
        return buf.value.decode()

    def ordering_report(self, recs):
        buf = C.create_string_buffer(1 << 20)
        agree = C.c_double()
        assert self.lib.ref_ordering_report(*self._records(recs), buf, _sz(1 << 20), C.byref(agree)) == 0
        return buf.value.decode(), agree.value

    def matrix_csv_write(self, a) -> str:
        a = _F(a)
        buf = C.create_string_buffer(1 << 20)
        assert self.lib.ref_matrix_csv_write(_p(a), _sz(a.shape[0]), _sz(a.shape[1]), buf, _sz(1 << 20)) == 0
        return buf.value.decode()

    def matrix_csv_read(self, text: str):
        out = np.zeros(1 << 16)
        m, n = _sz(0), _sz(0)
        self._status(self.lib.ref_matrix_csv_read(text.encode(), _p(out), _sz(out.size), C.byref(m), C.byref(n)))
        return out[: m.value * n.value].reshape((m.value, n.value), order="F")
