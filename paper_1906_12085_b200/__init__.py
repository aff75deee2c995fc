"""paper_1906_12085_b200 — B200-native FP64 PCA/SVD engine (svdkit drop-in).

The compute engine is libsvdk.so (hand-written sm_100a CUDA behind the C-ABI
in include/svdk.h). `svdkit` mirrors the reference svdkit API on numpy arrays;
`engine` exposes the device-pointer entry points for torch CUDA tensors.
"""
from . import errors
from ._lib import LIB_PATH, Context, load, nccl_unique_id
from .errors import DimensionError, EngineError, Error, FormatError, IoError, NumericalError, ParamError

__all__ = ["errors", "LIB_PATH", "Context", "load", "nccl_unique_id", "DimensionError", "Error",
           "NumericalError", "ParamError", "EngineError", "FormatError", "IoError", "svdkit", "engine",
           "cost_model", "csv_io", "idx_io", "bench_grid"]


def __getattr__(name):
    if name in ("svdkit", "engine", "cost_model", "csv_io", "idx_io", "bench_grid"):
        import importlib
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
