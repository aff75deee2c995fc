"""IDX image ingestion (reference idx_io.hpp, idx_io.cpp:24-107).

`parse_idx_images` validates the rank-3 unsigned-byte container through the
C-ABI (`svdk_idx_parse`, same checks / byte offsets as the reference);
`images_to_matrix` expands the pixels into the PCA input layout ON THE GPU
(`svdk_idx_to_matrix`: the 1-byte pixels cross PCIe, one sm_100a kernel writes
the count x (h*w) FP64 matrix, value = byte / 255 bit-identical to the
reference). `images_to_matrix_dev` does the same into a device buffer for
svdk_dev_pca (no host round trip of the doubles).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import IoError, ParamError


@dataclass
class IdxImageSet:
    """idx_io.hpp:13-19; pixels: count*height*width bytes, row-major per image."""
    count: int
    height: int
    width: int
    pixels: np.ndarray


def parse_idx_images(data: bytes) -> IdxImageSet:
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    dims = (C.c_uint64 * 3)()
    off = C.c_uint64(0)
    code = _lib.load().svdk_idx_parse(buf.ctypes.data if buf.size else None, buf.size, dims,
                                      C.byref(off))
    _lib.check(code, off.value)
    return IdxImageSet(int(dims[0]), int(dims[1]), int(dims[2]), buf[16:].copy())


def load_idx_file(path: str) -> IdxImageSet:
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    return parse_idx_images(data)


def images_to_matrix(s: IdxImageSet, ctx: _lib.Context | None = None) -> np.ndarray:
    """idx_io.cpp:84-94 on the GPU: count x (h*w), rows are examples."""
    ctx = ctx or _lib.default_context()
    p = s.height * s.width
    px = np.ascontiguousarray(s.pixels, dtype=np.uint8)
    if px.size != s.count * p:
        raise ParamError("images_to_matrix: pixel buffer does not match the dimensions")
    out = np.empty((s.count, p), dtype=np.float64, order="F")
    if out.size:
        _lib.check(_lib.load().svdk_idx_to_matrix(ctx.handle, px.ctypes.data, s.count, p,
                                                  out.ctypes.data))
    return out


def images_to_matrix_dev(ctx: _lib.Context, pixels_ptr: int, count: int, pixels_per_image: int,
                         out_ptr: int, ldo: int) -> None:
    """Device-buffer variant (svdk_dev_idx_to_matrix) on the context's stream."""
    _lib.check(_lib.load().svdk_dev_idx_to_matrix(ctx.handle, C.c_void_p(pixels_ptr), count,
                                                  pixels_per_image, C.c_void_p(out_ptr), ldo))


def image_as_matrix(s: IdxImageSet, index: int) -> np.ndarray:
    """idx_io.cpp:96-107: one image as height x width in [0, 1] (host: a single image)."""
    if index < 0 or index >= s.count:
        raise ParamError(f"image index {index} out of range, have {s.count} images")
    p = s.height * s.width
    img = s.pixels[index * p:(index + 1) * p].reshape(s.height, s.width)
    return np.asfortranarray(img.astype(np.float64) / 255.0)
