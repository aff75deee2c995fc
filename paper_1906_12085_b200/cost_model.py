"""Modeled cost of one factorization (reference cost_model.hpp / cost_model.cpp:30-113).

Thin binding of `svdk_cost_model` (paper_1906_12085_b200/csrc/cost_model.cu),
which restates the paper's published flop / storage closed forms. Space is
counted in 8-byte entries with the input included; bytes = 8 x entries.
Domain violations (m >= n >= l >= 1, i >= 0 / 1) raise ParamError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib

TRUNCATED, RANDOMIZED, RANDOMIZED_PRACTICAL = 0, 1, 2
KRYLOV, KRYLOV_PRACTICAL, KRYLOV_PER_STEP = 3, 4, 5


@dataclass(frozen=True)
class CostEstimate:
    """cost_model.hpp:11-15"""
    flops: float = 0.0
    space_entries: float = 0.0
    space_bytes: float = 0.0


def _model(model: int, m: int, n: int, l: int = 0, i: int = 0) -> CostEstimate:
    for v in (m, n, l, i):
        if int(v) < 0:
            from .errors import ParamError
            raise ParamError("cost model: sizes must be non-negative")
    f, e, b = C.c_double(), C.c_double(), C.c_double()
    _lib.check(_lib.load().svdk_cost_model(model, int(m), int(n), int(l), int(i), C.byref(f),
                                           C.byref(e), C.byref(b)))
    return CostEstimate(f.value, e.value, b.value)


def truncated_cost(m: int, n: int) -> CostEstimate:
    return _model(TRUNCATED, m, n)


def randomized_cost(m: int, n: int, l: int, i: int) -> CostEstimate:
    return _model(RANDOMIZED, m, n, l, i)


def randomized_cost_practical(m: int, n: int) -> CostEstimate:
    return _model(RANDOMIZED_PRACTICAL, m, n)


def krylov_cost(m: int, n: int, l: int, i: int) -> CostEstimate:
    return _model(KRYLOV, m, n, l, i)


def krylov_cost_practical(m: int, n: int) -> CostEstimate:
    return _model(KRYLOV_PRACTICAL, m, n)


def krylov_cost_per_step(m: int, n: int, l: int, i: int) -> CostEstimate:
    return _model(KRYLOV_PER_STEP, m, n, l, i)
