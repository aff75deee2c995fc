"""CSV matrix / vector text format (reference csv_io.hpp, csv_io.cpp:13-133).

Host-side text handling around the GPU path (inputs for fit_pca, outputs of
the bench grid). Numbers are written in the reference's `format_double`
form — std::to_chars(double): the shortest digit string that round-trips,
printed in fixed or scientific notation, whichever is shorter (ties -> fixed)
— so files are byte-identical to the reference's.
"""
from __future__ import annotations

import math
from decimal import Decimal
from typing import Iterable, TextIO

import numpy as np

from .errors import FormatError, IoError


def format_double(value: float) -> str:
    """csv_io.cpp:13-17 (std::to_chars shortest round-trip)."""
    v = float(value)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0"
    # repr() yields the shortest round-trip digits (correctly rounded)
    t = Decimal(repr(abs(v))).normalize().as_tuple()
    digits = "".join(map(str, t.digits))
    k, x = len(digits), t.exponent  # value = digits * 10^x
    e = k - 1 + x                    # scientific exponent
    sci = digits[0] + ("." + digits[1:] if k > 1 else "") + "e" + ("-" if e < 0 else "+") + \
        f"{abs(e):02d}"
    if x >= 0:
        # an integer: fixed notation prints the double's exact value (same length)
        fixed = str(int(abs(v)))
    elif k + x > 0:
        fixed = digits[:k + x] + "." + digits[k + x:]
    else:
        fixed = "0." + "0" * (-x - k) + digits
    return sign + (fixed if len(fixed) <= len(sci) else sci)


_WS = " \t\r"


def _parse_field(field: str, line_no: int) -> float:
    t = field.strip(_WS)
    bad = FormatError(f"csv: bad number '{field}' on line {line_no}", line_no)
    # std::from_chars grammar: optional '-', digits / inf / nan; no '+', no spaces
    if not t or t[0] == "+" or any(ch.isspace() for ch in t) or "_" in t:
        raise bad
    low = t.lower().lstrip("-")
    if low.startswith("0x"):
        raise bad
    try:
        v = float(t)
    except ValueError:
        raise bad from None
    if not math.isfinite(v):
        raise bad
    return v


def read_matrix_csv(stream: TextIO) -> np.ndarray:
    """csv_io.cpp:49-88: headerless rows of comma-separated decimals; blank lines skipped."""
    rows = []
    for line_no, line in enumerate(stream.read().split("\n"), start=1):
        if not line.strip(_WS):
            continue
        row = [_parse_field(f, line_no) for f in line.split(",")]
        if rows and len(row) != len(rows[0]):
            raise FormatError(f"csv: line {line_no} has {len(row)} fields, expected {len(rows[0])}",
                              line_no)
        rows.append(row)
    if not rows:
        raise FormatError("csv: no data rows", 0)
    return np.asfortranarray(np.array(rows, dtype=np.float64))


def read_matrix_csv_file(path: str) -> np.ndarray:
    try:
        with open(path, "r", newline="") as f:
            return read_matrix_csv(f)
    except OSError as e:
        raise IoError(f"cannot open {path}") from e


def matrix_csv_text(a) -> str:
    a = np.asarray(a, dtype=np.float64)
    return "".join(",".join(format_double(x) for x in row) + "\n" for row in a)


def write_matrix_csv(a, stream: TextIO) -> None:
    """csv_io.cpp:99-109"""
    stream.write(matrix_csv_text(a))


def write_matrix_csv_file(a, path: str) -> None:
    try:
        with open(path, "w", newline="") as f:
            write_matrix_csv(a, f)
    except OSError as e:
        raise IoError(f"cannot open {path} for writing") from e


def write_vector_csv_file(values: Iterable[float], path: str) -> None:
    """csv_io.cpp:122-133: one value per line."""
    try:
        with open(path, "w", newline="") as f:
            f.write("".join(format_double(v) + "\n" for v in values))
    except OSError as e:
        raise IoError(f"cannot open {path} for writing") from e
