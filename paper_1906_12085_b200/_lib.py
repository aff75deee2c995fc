"""ctypes binding of libsvdk.so (the C-ABI declared in include/svdk.h).

The shared library is built in-tree (`make -C paper_1906_12085_b200` or
`__graft_entry__.build()`). There is no CPU fallback: if the library is
missing, or no sm_100 GPU is usable, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import EngineError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
# SVDK_LIB: development override (e.g. a -DSVDK_PROBES build under build/)
LIB_PATH = os.environ.get("SVDK_LIB") or os.path.join(_HERE, "libsvdk.so")

_i64 = C.c_int64
_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p
_ctxp = C.c_void_p
_ip64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes); mirrors include/svdk.h
SIGNATURES = {
    "svdk_ctx_create": (C.c_int, [C.c_int, C.POINTER(_ctxp)]),
    "svdk_ctx_destroy": (C.c_int, [_ctxp]),
    "svdk_ctx_set_stream": (C.c_int, [_ctxp, _vp]),
    "svdk_ctx_sync": (C.c_int, [_ctxp]),
    "svdk_last_error": (C.c_char_p, []),
    "svdk_last_residual": (C.c_double, []),
    "svdk_ctx_launches": (_i64, [_ctxp]),
    "svdk_ctx_last_sweeps": (C.c_int, [_ctxp]),
    "svdk_version": (C.c_char_p, []),
    "svdk_ctx_set_timing": (C.c_int, [_ctxp, C.c_int]),
    "svdk_ctx_timing_reset": (C.c_int, [_ctxp]),
    "svdk_ctx_timing_query": (C.c_int, [_ctxp, C.c_char_p, _ip64, _dp, _dp, _dp]),
    "svdk_ctx_timing_names": (C.c_int, [_ctxp, C.c_char_p, _i64]),
    "svdk_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "svdk_ctx_attach_nccl": (C.c_int, [_ctxp, C.c_char_p, C.c_int, C.c_int]),
    "svdk_host_group_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "svdk_host_group_destroy": (C.c_int, [_vp]),
    "svdk_ctx_attach_host_group": (C.c_int, [_ctxp, _vp, C.c_int]),
    "svdk_ctx_detach_comm": (C.c_int, [_ctxp]),
    "svdk_ctx_comm_info": (C.c_int, [_ctxp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "svdk_matmul": (C.c_int, [_ctxp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "svdk_matmul_transposed_left": (C.c_int, [_ctxp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "svdk_transpose": (C.c_int, [_ctxp, _vp, _i64, _i64, _vp]),
    "svdk_gram": (C.c_int, [_ctxp, _vp, _i64, _i64, _vp]),
    "svdk_frobenius_norm_sq": (C.c_int, [_ctxp, _vp, _i64, _i64, _dp]),
    "svdk_qr_thin": (C.c_int, [_ctxp, _vp, _i64, _i64, _vp, _vp, _ip64]),
    "svdk_eig_sym": (C.c_int, [_ctxp, _vp, _i64, C.c_int, _vp, _vp]),
    "svdk_gaussian_matrix": (C.c_int, [_i64, _i64, _u64, _vp]),
    "svdk_truncated_svd": (C.c_int, [_ctxp, _vp, _i64, _i64, _vp, _vp, _vp, _ip64]),
    "svdk_randomized_pca": (C.c_int, [_ctxp, _vp, _i64, _i64, _i64, _i64, _u64, _vp, _vp, _vp, _ip64]),
    "svdk_krylov_svd": (C.c_int, [_ctxp, _vp, _i64, _i64, _i64, _i64, _u64, _vp, _vp, _vp, _ip64]),
    "svdk_lanczos_svd": (C.c_int, [_ctxp, _vp, _i64, _i64, _i64, _u64, _vp, _vp, _vp, _ip64]),
    "svdk_compute_svd": (C.c_int, [_ctxp, _vp, _i64, _i64, C.c_int, _i64, _i64, _u64, _vp, _vp, _vp, _ip64]),
    "svdk_center": (C.c_int, [_ctxp, _vp, _i64, _i64, C.c_int, _vp, _vp]),
    "svdk_select_components": (C.c_int, [_ctxp, _vp, _i64, C.c_double, C.c_double, _ip64]),
    "svdk_fit_pca": (C.c_int, [_ctxp, _vp, _i64, _i64, C.c_int, C.c_int, _i64, _i64, _u64, C.c_int,
                               _vp, _vp, _dp, _vp, _ip64]),
    "svdk_residual_delta": (C.c_int, [_ctxp, _vp, _i64, _i64, _vp, _vp, _vp, _i64, _dp]),
    "svdk_dev_gemm": (C.c_int, [_ctxp, C.c_int, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64]),
    "svdk_dev_gram": (C.c_int, [_ctxp, _vp, _i64, _i64, _i64, _vp, _i64]),
    "svdk_dev_gemv_pair": (C.c_int, [_ctxp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "svdk_dev_eig_sym": (C.c_int, [_ctxp, _vp, _i64, _i64, C.c_int, _vp, _vp, _i64]),
    "svdk_dev_qr_thin": (C.c_int, [_ctxp, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _ip64]),
    "svdk_dev_pca": (C.c_int, [_ctxp, _vp, _i64, _i64, _i64, C.c_int, _i64, _i64, _u64, C.c_int,
                               C.c_double, _vp, _i64, _vp, _vp, _i64, _vp, _ip64, _ip64, _dp]),
    "svdk_dev_idx_to_matrix": (C.c_int, [_ctxp, _vp, _i64, _i64, _vp, _i64]),
    "svdk_cost_model": (C.c_int, [C.c_int, _u64, _u64, _u64, _u64, _dp, _dp, _dp]),
    "svdk_idx_parse": (C.c_int, [_vp, _u64, C.POINTER(_u64), C.POINTER(_u64)]),
    "svdk_idx_to_matrix": (C.c_int, [_ctxp, _vp, _i64, _i64, _vp]),
    "svdk_synth_fill": (C.c_int, [_u64, C.c_int, C.c_int, _i64, _i64, _i64, _i64, _vp, _i64]),
    "svdk_synth_add_noise": (C.c_int, [_u64, _i64, _i64, _i64, _i64, C.c_double, _vp, _i64]),
    "svdk_synth_mixing": (C.c_int, [_i64, _vp, _i64, _vp, _u64, _vp, _i64, _dp]),
    "svdk_dev_synth_fill": (C.c_int, [_ctxp, _u64, C.c_int, C.c_int, _i64, _i64, _i64, _i64, _vp, _i64]),
    "svdk_dev_synth_add_noise": (C.c_int, [_ctxp, _u64, _i64, _i64, _i64, _i64, C.c_double, _vp, _i64]),
}

_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load libsvdk.so once; raise EngineError if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise EngineError(
                    f"{LIB_PATH} not found: build the CUDA engine first "
                    "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback."
                )
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def check(code: int, offset: int = 0) -> None:
    if code != 0:
        lib = load()
        msg = lib.svdk_last_error().decode(errors="replace")
        raise_for_status(code, msg, lib.svdk_last_residual(), offset)


class Context:
    """One GPU, one stream, one device memory pool (svdk_ctx)."""

    def __init__(self, device: int = 0):
        lib = load()
        h = _ctxp()
        check(lib.svdk_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: int) -> None:
        check(load().svdk_ctx_set_stream(self._h, _vp(stream_ptr)))

    def sync(self) -> None:
        check(load().svdk_ctx_sync(self._h))

    def launches(self) -> int:
        return int(load().svdk_ctx_launches(self._h))

    def last_sweeps(self) -> int:
        return int(load().svdk_ctx_last_sweeps(self._h))

    def set_timing(self, enable: bool) -> None:
        check(load().svdk_ctx_set_timing(self._h, 1 if enable else 0))

    def timing_reset(self) -> None:
        check(load().svdk_ctx_timing_reset(self._h))

    def timing(self, name: str | None = None) -> dict:
        """{count, ms, flops, bytes} summed over records named `name` (None = all)."""
        cnt, ms, fl, by = C.c_int64(0), C.c_double(0), C.c_double(0), C.c_double(0)
        check(load().svdk_ctx_timing_query(self._h, name.encode() if name else None, C.byref(cnt), C.byref(ms),
                                           C.byref(fl), C.byref(by)))
        return {"count": cnt.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}

    def timing_names(self) -> list:
        buf = C.create_string_buffer(4096)
        check(load().svdk_ctx_timing_names(self._h, buf, 4096))
        return [x for x in buf.value.decode().split(",") if x]

    def attach_nccl(self, unique_id: bytes, rank: int, world: int) -> None:
        check(load().svdk_ctx_attach_nccl(self._h, unique_id, int(rank), int(world)))

    def attach_host_group(self, group: "HostGroup", rank: int) -> None:
        check(load().svdk_ctx_attach_host_group(self._h, group.handle, int(rank)))

    def detach_comm(self) -> None:
        check(load().svdk_ctx_detach_comm(self._h))

    def comm_info(self) -> tuple:
        r, w = C.c_int(0), C.c_int(0)
        check(load().svdk_ctx_comm_info(self._h, C.byref(r), C.byref(w)))
        return r.value, w.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            load().svdk_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostGroup:
    """In-process host-staged collective group (svdk_host_group_*): `world`
    contexts driven by host threads act as the ranks of a row-sharded call."""

    def __init__(self, world: int):
        h = _vp()
        check(load().svdk_host_group_create(int(world), C.byref(h)))
        self.handle = h
        self.world = world

    def close(self) -> None:
        if getattr(self, "handle", None):
            load().svdk_host_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(load().svdk_nccl_unique_id(buf))
    return buf.raw


_default = {}


def default_context(device: int = 0) -> Context:
    ctx = _default.get(device)
    if ctx is None:
        ctx = Context(device)
        _default[device] = ctx
    return ctx
