"""Benchmark grid on the GPU (reference bench.hpp, bench.cpp:50-244).

Reproduces the paper's experiment shape: the cross product of row / column
sizes, each cell run for every selected method on Gaussian test matrices,
timed, checked with the relative residual delta and annotated with the
paper's cost model. The factorisations and delta run on the B200 engine
(svdkit.compute_svd / residual_delta); the text outputs (CSV, ordering report)
are byte-compatible with the reference's.

    python -m paper_1906_12085_b200.bench_grid --rows 2000,4000 --cols 100,200 \\
        --methods truncated,randomized,krylov --repeats 3 --csv grid.csv --report

Per cell and trial the input is gaussian_matrix(m, n, seed + trial) (host
sampler, bit-identical to the reference, outside the timed region) and the
sketch methods get seed + 0x9e3779b97f4a7c15 + trial (bench.cpp:22-24,
116-119). The timed region is one compute_svd call, host buffers in and out,
like the reference's steady_clock bracket (bench.cpp:121-125).
"""
from __future__ import annotations

import argparse
import math
import sys
import time
from dataclasses import dataclass, field
from typing import List, Tuple

from . import cost_model, svdkit
from .csv_io import format_double
from .errors import IoError, ParamError
from .svdkit import MethodParams, RngSeed, SvdMethod, method_name

METHOD_SEED_OFFSET = 0x9E3779B97F4A7C15
_U64 = (1 << 64) - 1


@dataclass
class BenchConfig:
    """bench.hpp:15-24"""
    row_sizes: List[int] = field(default_factory=list)
    col_sizes: List[int] = field(default_factory=list)
    methods: List[SvdMethod] = field(default_factory=list)
    repeats: int = 10
    seed: RngSeed = RngSeed(42)
    l_fraction: float = 0.5
    iterations: int = 1
    memory_cap_bytes: float = 2.0 * 1024 * 1024 * 1024


@dataclass
class BenchRecord:
    """bench.hpp:28-38"""
    method: SvdMethod = SvdMethod.Truncated
    m: int = 0
    n: int = 0
    repeats: int = 0
    mean_seconds: float = 0.0
    std_seconds: float = 0.0
    delta: float = 0.0
    model_flops: float = 0.0
    model_space_bytes: float = 0.0


@dataclass
class SkippedCell:
    method: SvdMethod
    m: int
    n: int
    reason: str


@dataclass
class GridResult:
    records: List[BenchRecord] = field(default_factory=list)
    skipped: List[SkippedCell] = field(default_factory=list)


def _validate(cfg: BenchConfig) -> None:
    """bench.cpp:26-48"""
    if not cfg.row_sizes or not cfg.col_sizes:
        raise ParamError("bench: empty grid")
    if not cfg.methods:
        raise ParamError("bench: no methods selected")
    if cfg.repeats < 1:
        raise ParamError("bench: repeats must be >= 1")
    if not (cfg.l_fraction > 0.0 and cfg.l_fraction <= 1.0):
        raise ParamError("bench: l_fraction must be in (0, 1]")
    for m in cfg.row_sizes:
        for n in cfg.col_sizes:
            if m < n:
                raise ParamError(f"bench: grid cell {m}x{n} violates m >= n")


def expand_grid(cfg: BenchConfig) -> List[Tuple[int, int]]:
    """bench.cpp:52-66: cells sorted m ascending, then n ascending."""
    _validate(cfg)
    return [(m, n) for m in sorted(cfg.row_sizes) for n in sorted(cfg.col_sizes)]


def sketch_width_for(cfg: BenchConfig, n: int) -> int:
    """bench.cpp:68-72: clamp(ceil(l_fraction * n), 1, n)."""
    return min(max(int(math.ceil(cfg.l_fraction * float(n))), 1), n)


def _cost(method: SvdMethod, m: int, n: int, l: int, i: int) -> cost_model.CostEstimate:
    if method == SvdMethod.Truncated:
        return cost_model.truncated_cost(m, n)
    if method == SvdMethod.Randomized:
        return cost_model.randomized_cost(m, n, l, i)
    if method == SvdMethod.Krylov:
        return cost_model.krylov_cost(m, n, l, i)
    raise ParamError(f"bench: no published cost model for {method_name(method)}")


def run_grid(cfg: BenchConfig, progress=None) -> GridResult:
    """bench.cpp:74-146 with the factorisation and delta on the GPU."""
    cells = expand_grid(cfg)
    methods = sorted(set(SvdMethod(x) for x in cfg.methods), key=method_name)
    result = GridResult()
    for m, n in cells:
        matrix_bytes = 8.0 * float(m) * float(n)
        l = sketch_width_for(cfg, n)
        for method in methods:
            if matrix_bytes > cfg.memory_cap_bytes:
                result.skipped.append(SkippedCell(
                    method, m, n, f"matrix needs {matrix_bytes:f} bytes, cap is {cfg.memory_cap_bytes:f}"))
                continue
            if method == SvdMethod.Krylov and (cfg.iterations + 1) * l > m:
                result.skipped.append(SkippedCell(
                    method, m, n, f"krylov block width {(cfg.iterations + 1) * l} exceeds m = {m}"))
                continue
            cost = _cost(method, m, n, l, cfg.iterations)
            seconds, delta_sum = [], 0.0
            for trial in range(cfg.repeats):
                a = svdkit.gaussian_matrix(m, n, RngSeed((cfg.seed.value + trial) & _U64))
                params = MethodParams(l, cfg.iterations,
                                      RngSeed((cfg.seed.value + METHOD_SEED_OFFSET + trial) & _U64))
                t0 = time.perf_counter()
                s = svdkit.compute_svd(a, method, params)
                seconds.append(time.perf_counter() - t0)
                delta_sum += svdkit.residual_delta(a, s)
            mean = sum(seconds) / cfg.repeats
            var = 0.0
            if cfg.repeats > 1:
                var = sum((t - mean) * (t - mean) for t in seconds) / (cfg.repeats - 1)
            rec = BenchRecord(method, m, n, cfg.repeats, mean, math.sqrt(var), delta_sum / cfg.repeats,
                              cost.flops, cost.space_bytes)
            result.records.append(rec)
            if progress:
                progress(rec)
    return result


CSV_HEADER = "method,m,n,repeats,mean_seconds,std_seconds,delta,model_flops,model_space_bytes\n"


def to_csv(records: List[BenchRecord]) -> str:
    """bench.cpp:148-158"""
    out = [CSV_HEADER]
    for r in records:
        out.append(f"{method_name(r.method)},{r.m},{r.n},{r.repeats},{format_double(r.mean_seconds)},"
                   f"{format_double(r.std_seconds)},{format_double(r.delta)},"
                   f"{format_double(r.model_flops)},{format_double(r.model_space_bytes)}\n")
    return "".join(out)


def write_csv_file(records: List[BenchRecord], path: str) -> None:
    try:
        with open(path, "w", newline="\n") as f:
            f.write(to_csv(records))
    except OSError as e:
        raise IoError(f"cannot open {path} for writing") from e


@dataclass
class OrderingCell:
    m: int = 0
    n: int = 0
    by_seconds: List[SvdMethod] = field(default_factory=list)
    by_flops: List[SvdMethod] = field(default_factory=list)
    agree: bool = False


@dataclass
class OrderingReport:
    cells: List[OrderingCell] = field(default_factory=list)
    agreement: float = 0.0


def summarize_ordering(records: List[BenchRecord]) -> OrderingReport:
    """bench.cpp:172-212: per-cell rankings by measured time and by modeled flops."""
    cells = {}
    for r in records:
        cells.setdefault((r.m, r.n), []).append(r)
    report = OrderingReport()
    agreeing = 0
    for (m, n) in sorted(cells):
        recs = cells[(m, n)]
        by_s = [r.method for r in sorted(recs, key=lambda r: (r.mean_seconds, method_name(r.method)))]
        by_f = [r.method for r in sorted(recs, key=lambda r: (r.model_flops, method_name(r.method)))]
        cell = OrderingCell(m, n, by_s, by_f, by_s == by_f)
        agreeing += cell.agree
        report.cells.append(cell)
    report.agreement = agreeing / len(report.cells) if report.cells else 0.0
    return report


def format_report(report: OrderingReport) -> str:
    """bench.cpp:214-242 (fixed-width table; lines capped at 159 characters like the C buffer)."""
    out = ["cell            measured (fast->slow)              modeled (cheap->costly)"
           "            agree\n"]
    for c in report.cells:
        measured = " < ".join(method_name(x) for x in c.by_seconds)
        modeled = " < ".join(method_name(x) for x in c.by_flops)
        line = f"{c.m:6d}x{c.n:<6d}  {measured:<34s} {modeled:<34s} {'yes' if c.agree else 'NO'}\n"
        out.append(line[:159])
    out.append(f"ranking agreement: {report.agreement:.2f}\n"[:63])
    return "".join(out)


def _sizes(text: str) -> List[int]:
    return [int(x) for x in text.split(",") if x.strip()]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--rows", required=True, help="comma-separated m values")
    ap.add_argument("--cols", required=True, help="comma-separated n values")
    ap.add_argument("--methods", default="truncated,randomized,krylov")
    ap.add_argument("--repeats", type=int, default=10)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--l-fraction", type=float, default=0.5)
    ap.add_argument("--iterations", type=int, default=1)
    ap.add_argument("--memory-cap-bytes", type=float, default=2.0 * 1024 ** 3)
    ap.add_argument("--csv", default=None, help="write the records here (default: stdout)")
    ap.add_argument("--report", action="store_true", help="print the method-ordering report")
    args = ap.parse_args(argv)
    methods = []
    for name in args.methods.split(","):
        mth = svdkit.method_from_name(name.strip())
        if mth is None:
            raise ParamError(f"bench: unknown method '{name}'")
        methods.append(mth)
    cfg = BenchConfig(_sizes(args.rows), _sizes(args.cols), methods, args.repeats, RngSeed(args.seed),
                      args.l_fraction, args.iterations, args.memory_cap_bytes)
    res = run_grid(cfg, progress=lambda r: print(
        f"{method_name(r.method):>10s} {r.m:>8d}x{r.n:<6d} {r.mean_seconds * 1e3:10.3f} ms  "
        f"delta {r.delta:.3e}", file=sys.stderr))
    for s in res.skipped:
        print(f"skipped {method_name(s.method)} {s.m}x{s.n}: {s.reason}", file=sys.stderr)
    if args.csv:
        write_csv_file(res.records, args.csv)
    else:
        sys.stdout.write(to_csv(res.records))
    if args.report:
        sys.stdout.write(format_report(summarize_ordering(res.records)))
    return 0


if __name__ == "__main__":
    sys.exit(main())
