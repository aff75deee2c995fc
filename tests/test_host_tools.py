"""Parity of the host-side tools around the GPU path with
the reference compiled in place (oracle/_ref): cost model, CSV number format
and parsing, IDX header validation, bench-grid expansion / CSV / ordering
report. CPU only — the C-ABI parts here (svdk_cost_model, svdk_idx_parse)
touch no GPU. GPU parts (images_to_matrix, run_grid) are in test_gpu_tools.py.
"""
import io
import math
import struct

import numpy as np
import pytest

from paper_1906_12085_b200 import bench_grid, cost_model, csv_io, idx_io
from paper_1906_12085_b200.errors import FormatError, ParamError
from paper_1906_12085_b200.svdkit import SvdMethod


@pytest.fixture(scope="module")
def rt():
    from oracle.pyoracle import RefTools, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefTools()


# ---------------------------------------------------------------- cost model
COST_CASES = [(1, 1, 1, 0), (10, 4, 2, 1), (60000, 784, 392, 1), (200000, 1024, 1024, 2),
              (8388608, 1024, 512, 3), (65536, 4096, 4096, 3), (5, 5, 5, 7), (1000, 10, 3, 0)]


@pytest.mark.parametrize("m,n,l,i", COST_CASES)
def test_cost_model_matches_reference(rt, m, n, l, i):
    fns = {
        cost_model.TRUNCATED: lambda: cost_model.truncated_cost(m, n),
        cost_model.RANDOMIZED: lambda: cost_model.randomized_cost(m, n, l, i),
        cost_model.RANDOMIZED_PRACTICAL: lambda: cost_model.randomized_cost_practical(m, n),
        cost_model.KRYLOV: lambda: cost_model.krylov_cost(m, n, l, i),
        cost_model.KRYLOV_PRACTICAL: lambda: cost_model.krylov_cost_practical(m, n),
        cost_model.KRYLOV_PER_STEP: lambda: cost_model.krylov_cost_per_step(m, n, l, i),
    }
    for model, fn in fns.items():
        try:
            want = rt.cost(model, m, n, l, i)
        except Exception as e:  # domain error in the reference -> ParamError here
            assert getattr(e, "code", None) == 2
            with pytest.raises(ParamError):
                fn()
            continue
        got = fn()
        assert (got.flops, got.space_entries, got.space_bytes) == want, (model, got, want)
        assert got.space_bytes == 8.0 * got.space_entries


@pytest.mark.parametrize("args", [(3, 4, 1, 1), (10, 4, 5, 1), (10, 4, 0, 1)])
def test_cost_model_domain_errors(rt, args):
    m, n, l, i = args
    for model in (cost_model.RANDOMIZED, cost_model.KRYLOV, cost_model.KRYLOV_PER_STEP):
        with pytest.raises(Exception):
            rt.cost(model, m, n, l, i)
        with pytest.raises(ParamError):
            cost_model._model(model, m, n, l, i)
    with pytest.raises(ParamError):  # krylov needs i >= 1
        cost_model.krylov_cost(10, 4, 2, 0)


# ---------------------------------------------------------------- CSV
SPECIAL = [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e-4, 1e-5, 0.0001234, 123.0, 1e15, 1e16, 1e17, 1e21, 1e22,
           123456789012345680.0, 1.2345678901234567e-7, 5e-324, 2.2250738585072014e-308,
           1.7976931348623157e308, 3.0, 1.5e300, 299792458.0, 6.02214076e23, 2.5, 0.30000000000000004,
           100.0, 1000000.0, 1e7, 12345678.9, 0.001, 0.01]


def test_format_double_matches_reference(rt):
    rng = np.random.default_rng(5)
    vals = list(SPECIAL) + [-v for v in SPECIAL]
    vals += list(rng.standard_normal(300) * 10.0 ** rng.integers(-30, 30, 300))
    vals += list(rng.integers(-10 ** 9, 10 ** 9, 100).astype(float))
    vals += list(np.frombuffer(rng.bytes(8 * 400), dtype=np.float64))
    for v in vals:
        v = float(v)
        if not math.isfinite(v):
            continue
        assert csv_io.format_double(v) == rt.format_double(v), v


def test_matrix_csv_write_matches_reference(rt):
    rng = np.random.default_rng(1)
    a = np.asfortranarray(rng.standard_normal((7, 5)) * 10.0 ** rng.integers(-8, 8, (7, 5)))
    assert csv_io.matrix_csv_text(a) == rt.matrix_csv_write(a)


CSV_GOOD = ["1,2,3\n4,5,6\n", "1.5, -2e-3 ,\t7\r\n\n  \n8,9,10", " 0.25\n-0\n1e300\n", ".5,5.\n1,2\n",
            "1,2\n3,4"]
CSV_BAD = ["", "\n\n", "1,2\n3\n", "1,,2\n", "1,abc\n", "nan,1\n", "1e999\n", "+1,2\n", "0x10\n",
           "1 2\n", "1_0\n", "inf\n"]


@pytest.mark.parametrize("text", CSV_GOOD)
def test_read_matrix_csv_matches_reference(rt, text):
    want = rt.matrix_csv_read(text)
    got = csv_io.read_matrix_csv(io.StringIO(text))
    assert got.shape == want.shape
    assert np.array_equal(got, want)


@pytest.mark.parametrize("text", CSV_BAD)
def test_read_matrix_csv_errors_match_reference(rt, text):
    with pytest.raises(Exception) as ref_err:
        rt.matrix_csv_read(text)
    assert ref_err.value.code == 8
    with pytest.raises(FormatError) as err:
        csv_io.read_matrix_csv(io.StringIO(text))
    assert err.value.offset() == ref_err.value.offset  # the line number


def test_csv_file_round_trip(tmp_path):
    rng = np.random.default_rng(2)
    a = rng.standard_normal((6, 4))
    p = str(tmp_path / "a.csv")
    csv_io.write_matrix_csv_file(a, p)
    assert np.array_equal(csv_io.read_matrix_csv_file(p), a)  # shortest round-trip is exact
    csv_io.write_vector_csv_file([0.5, 1e-7], str(tmp_path / "v.csv"))
    assert open(tmp_path / "v.csv").read() == "0.5\n1e-07\n"


# ---------------------------------------------------------------- IDX
def idx_bytes(count, h, w, payload=None, magic=0x00000803, extra=b""):
    rng = np.random.default_rng(count * 131 + h * 7 + w)
    if payload is None:
        payload = rng.integers(0, 256, count * h * w, dtype=np.uint8).tobytes()
    return struct.pack(">IIII", magic, count, h, w) + payload + extra


IDX_BAD = [
    b"",                                   # short header
    b"\x00\x00\x08\x03\x00",               # short header
    idx_bytes(2, 3, 3, magic=0x00000801),  # wrong magic
    idx_bytes(0, 3, 3, payload=b""),       # zero dimension
    idx_bytes(2, 0, 3, payload=b""),
    struct.pack(">IIII", 0x803, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF),  # product overflow (on 64 bit: no)
    idx_bytes(2, 3, 3)[:-1],               # truncated payload
    idx_bytes(2, 3, 3, extra=b"\x00"),     # trailing bytes
]


def test_idx_parse_valid_matches_reference(rt):
    for dims in [(1, 1, 1), (3, 28, 28), (10, 5, 7)]:
        data = idx_bytes(*dims)
        assert rt.idx_parse(data) == dims
        s = idx_io.parse_idx_images(data)
        assert (s.count, s.height, s.width) == dims
        assert s.pixels.tobytes() == data[16:]


@pytest.mark.parametrize("k", range(len(IDX_BAD)))
def test_idx_parse_errors_match_reference(rt, k):
    data = IDX_BAD[k]
    with pytest.raises(Exception) as ref_err:
        rt.idx_parse(data)
    assert ref_err.value.code == 8
    with pytest.raises(FormatError) as err:
        idx_io.parse_idx_images(data)
    assert err.value.offset() == ref_err.value.offset


def test_image_as_matrix_matches_reference(rt):
    data = idx_bytes(4, 6, 5)
    s = idx_io.parse_idx_images(data)
    for i in range(4):
        assert np.array_equal(idx_io.image_as_matrix(s, i), rt.image_as_matrix(data, i))
    with pytest.raises(ParamError):
        idx_io.image_as_matrix(s, 4)


# ---------------------------------------------------------------- bench grid text
def test_expand_grid_and_sketch_width_match_reference(rt):
    cfg = bench_grid.BenchConfig([4000, 1000, 2000], [300, 100], [SvdMethod.Truncated])
    assert bench_grid.expand_grid(cfg) == rt.expand_grid([4000, 1000, 2000], [300, 100])
    for frac in (0.5, 0.1, 1.0, 0.333, 1e-9):
        for n in (1, 2, 3, 10, 784, 1001):
            cfg.l_fraction = frac
            assert bench_grid.sketch_width_for(cfg, n) == rt.sketch_width_for(frac, n)
    with pytest.raises(ParamError):
        bench_grid.expand_grid(bench_grid.BenchConfig([10], [20], [SvdMethod.Truncated]))
    with pytest.raises(Exception):
        rt.expand_grid([10], [20])
    for bad in (bench_grid.BenchConfig([], [2], [SvdMethod.Truncated]),
                bench_grid.BenchConfig([4], [2], []),
                bench_grid.BenchConfig([4], [2], [SvdMethod.Truncated], repeats=0),
                bench_grid.BenchConfig([4], [2], [SvdMethod.Truncated], l_fraction=0.0)):
        with pytest.raises(ParamError):
            bench_grid.expand_grid(bad)


def synthetic_records():
    rng = np.random.default_rng(9)
    recs = []
    for m, n in [(1000, 100), (2000, 100), (2000, 200), (4000, 300)]:
        for meth in (SvdMethod.Krylov, SvdMethod.Randomized, SvdMethod.Truncated):
            l = max(1, n // 2)
            c = {SvdMethod.Truncated: cost_model.truncated_cost(m, n),
                 SvdMethod.Randomized: cost_model.randomized_cost(m, n, l, 1),
                 SvdMethod.Krylov: cost_model.krylov_cost(m, n, l, 1)}[meth]
            recs.append(bench_grid.BenchRecord(meth, m, n, 3, float(rng.uniform(1e-4, 1e-1)),
                                               float(rng.uniform(0, 1e-3)), float(rng.uniform(1e-16, 1e-13)),
                                               c.flops, c.space_bytes))
    # a tie on time resolved by method name, and a record with zero std
    recs.append(bench_grid.BenchRecord(SvdMethod.Truncated, 5000, 10, 1, 0.5, 0.0, 0.0, 1.0, 8.0))
    recs.append(bench_grid.BenchRecord(SvdMethod.Randomized, 5000, 10, 1, 0.5, 0.0, 0.0, 2.0, 8.0))
    return recs


def as_tuples(recs):
    return [(int(r.method), r.m, r.n, r.repeats, r.mean_seconds, r.std_seconds, r.delta, r.model_flops,
             r.model_space_bytes) for r in recs]


def test_bench_csv_matches_reference(rt):
    recs = synthetic_records()
    assert bench_grid.to_csv(recs) == rt.bench_csv(as_tuples(recs))
    assert bench_grid.to_csv([]) == rt.bench_csv([]) == bench_grid.CSV_HEADER


def test_ordering_report_matches_reference(rt):
    recs = synthetic_records()
    text, agree = rt.ordering_report(as_tuples(recs))
    rep = bench_grid.summarize_ordering(recs)
    assert rep.agreement == agree
    assert bench_grid.format_report(rep) == text
    empty_text, empty_agree = rt.ordering_report([])
    assert bench_grid.format_report(bench_grid.summarize_ordering([])) == empty_text
    assert empty_agree == 0.0


def test_lanczos_has_no_published_cost_model():
    with pytest.raises(ParamError):
        bench_grid._cost(SvdMethod.Lanczos, 10, 5, 2, 1)


# ---------------------------------------------------------------- the C++ facade
TOOL_RECORDS = [  # facade/tools_test.cpp::records()
    (0, 1000, 100, 3, 0.012, 0.0005, 1e-15, 2.0e7, 8.0e5),
    (1, 1000, 100, 3, 0.004, 0.0001, 3.5e-3, 1.1e7, 6.4e5),
    (2, 1000, 100, 3, 0.007, 0.0, 2.5e-4, 9.9e10, 1.2e6),
    (0, 4000, 300, 1, 0.25, 0.0, 0.0, 7.2e8, 2.0e7),
    (1, 4000, 300, 1, 0.25, 0.0, 0.5, 3.3e8, 1.5e7),
]


def tool_idx(magic, c, h, w, payload, extra=0):
    return struct.pack(">IIII", magic, c, h, w) + bytes(((k * 7 + 3) & 255) for k in range(payload + extra))


def test_facade_tools_host_match_reference(rt):
    """facade/tools_test host (C++ API over libsvdkit.so, no GPU) vs the reference."""
    import os
    import subprocess
    from tests.conftest import ROOT
    exe = os.path.join(ROOT, "facade", "tools_test")
    if not os.path.exists(exe):
        pytest.skip("facade not built")
    out = subprocess.run([exe, "host"], capture_output=True, text=True, timeout=60, check=True).stdout
    body, rest = out.split("--csv--\n")
    csv_text, rest = rest.split("--report--\n")
    report_text = rest.split("--end--\n")[0]
    csv_cases = ["1,2\n3\n", "1,x\n", "", "1,2\n\n3,nan\n"]
    idx_cases = [tool_idx(0x803, 3, 4, 5, 60), tool_idx(0x803, 1, 1, 1, 1), bytes(7),
                 tool_idx(0x801, 3, 4, 5, 60), tool_idx(0x803, 0, 4, 5, 0), tool_idx(0x803, 3, 4, 5, 59),
                 tool_idx(0x803, 3, 4, 5, 60, 2)]
    csv_k = 0
    cells, widths = [], []
    seen = set()
    for line in body.splitlines():
        f = line.split()
        seen.add(f[0])
        if f[0] == "cost":
            model, m, n, l, i = map(int, f[1:6])
            try:
                want = rt.cost(model, m, n, l, i)
            except Exception:
                assert f[6] == "ParamError", line
                continue
            assert tuple(float.fromhex(x) for x in f[6:9]) == want, line
        elif f[0] == "fmt":
            assert f[2] == rt.format_double(float.fromhex(f[1])), line
        elif f[0] == "csv":
            try:
                rt.matrix_csv_read(csv_cases[csv_k])
                assert f[1] == "ok", line
            except Exception as e:
                assert f[1:] == ["FormatError", str(e.offset)], line
            csv_k += 1
        elif f[0] == "csvrt":
            a = rt.matrix_csv_read("1.5, -2e-3\n\n 7,8\r\n")
            assert line.split(" ", 3)[3] + "\n" == rt.matrix_csv_write(a).split("\n")[0] + "\n"
        elif f[0] == "idx":
            data = idx_cases[int(f[1])]
            try:
                c, h, w = rt.idx_parse(data)
            except Exception as e:
                assert f[2:] == ["FormatError", str(e.offset)], line
                continue
            assert list(map(int, f[2:5])) == [c, h, w]
            assert float.fromhex(f[5]) == rt.image_as_matrix(data, c - 1)[h - 1, 0]
        elif f[0] == "cell":
            cells.append((int(f[1]), int(f[2])))
        elif f[0] == "width":
            widths.append((int(f[1]), int(f[2])))
    assert {"cost", "fmt", "csv", "idx", "cell", "width"} <= seen and csv_k == len(csv_cases)
    assert cells == rt.expand_grid([4000, 1000], [300, 100])
    assert widths == [(n, rt.sketch_width_for(0.5, n)) for n in (1, 3, 784, 1001)]
    assert csv_text == rt.bench_csv(TOOL_RECORDS)
    assert report_text == rt.ordering_report(TOOL_RECORDS)[0]


# --------------------------------------------------------------------------- SYRK work tables (host logic)
def _syrk_table(tiles, rows, ctas, weight):
    import ctypes as C
    from paper_1906_12085_b200 import _lib
    lib = C.CDLL(_lib.LIB_PATH)
    lib.svdk_debug_syrk_line.restype = C.c_longlong
    lib.svdk_debug_syrk_line.argtypes = [C.c_int, C.c_longlong, C.c_int, C.c_int, C.POINTER(C.c_longlong), C.c_longlong]
    need = lib.svdk_debug_syrk_line(tiles, rows, ctas, weight, None, 0)
    if need <= 0:
        return None
    buf = (C.c_longlong * need)()
    assert lib.svdk_debug_syrk_line(tiles, rows, ctas, weight, buf, need) == need
    t = list(buf)
    units, n_tiles = t[0], tiles * (tiles + 1) // 2
    utab = [tuple(t[1 + 3 * u:4 + 3 * u]) for u in range(units)]
    o = 1 + 3 * units
    cfirst, tfirst, clist = t[o:o + ctas + 1], t[o + ctas + 1:o + ctas + 1 + n_tiles + 1], t[o + ctas + n_tiles + 2:]
    return utab, cfirst, tfirst, clist


def _check_syrk_table(tiles, rows, ctas, table, slack_steps):
    utab, cfirst, tfirst, clist = table
    units, n_tiles = len(utab), tiles * (tiles + 1) // 2
    assert len(tfirst) == n_tiles + 1 and cfirst[0] == 0 and cfirst[-1] == units and tfirst[-1] == units
    assert sorted(clist) == list(range(units))  # every unit runs on exactly one CTA
    assert all(a <= b for a, b in zip(cfirst, cfirst[1:]))
    diag = {tj * (tj + 1) // 2 + tj for tj in range(tiles)}
    for tile in range(n_tiles):  # a tile's pieces are contiguous in the table, in k order, and cover [0, K)
        pieces = utab[tfirst[tile]:tfirst[tile + 1]]
        assert pieces and all(p[0] == tile for p in pieces)
        assert pieces[0][1] == 0 and pieces[-1][2] == rows
        assert all(a[2] == b[1] and a[2] % 16 == 0 for a, b in zip(pieces, pieces[1:]))
        assert all(p[2] > p[1] for p in pieces)
    loads = []
    for b in range(ctas):
        w = 0
        for u in clist[cfirst[b]:cfirst[b + 1]]:
            tile, k0, k1 = utab[u]
            w += -(-(k1 - k0) // 16) * (19 if tile in diag else 32)
        loads.append(w)
    busy = [w for w in loads if w]
    mean = sum(busy) / len(busy)
    assert max(busy) - mean <= 32 * slack_steps and mean - min(busy) <= 32 * slack_steps, (max(busy), mean, min(busy))
    return loads


@pytest.mark.parametrize("tiles,rows,ctas", [(8, 8388608, 148), (8, 200000, 148), (32, 65536, 148), (16, 500000, 148),
                                             (2, 32768, 148), (1, 40000, 148), (3, 33001, 148), (8, 1 << 20, 7)])
def test_syrk_work_line_table(tiles, rows, ctas):
    """build_syrk_line (csrc/gemm_f64.cu): every upper tile's k range [0, K) is covered exactly once by
    contiguous pieces in piece order, a tile's pieces and a CTA's pieces are contiguous in the table, and the
    CTAs' weights (32 per full k-step, 19 per diagonal one) are equal to within one k-step per piece."""
    table = _syrk_table(tiles, rows, ctas, 0)
    utab, cfirst, tfirst, clist = table
    assert clist == list(range(len(utab)))  # the line: consecutive units per CTA
    assert sorted(u[0] for u in utab) == [u[0] for u in utab]
    pieces_max = max(cfirst[b + 1] - cfirst[b] for b in range(ctas))
    _check_syrk_table(tiles, rows, ctas, table, pieces_max + 1)


@pytest.mark.parametrize("tiles,rows,ctas", [(8, 8388608, 148), (8, 200000, 148), (8, 1 << 20, 148), (4, 65536, 148),
                                             (7, 300000, 148)])
def test_syrk_lockstep_table(tiles, rows, ctas):
    """build_syrk_lockstep: the tiles x S k-chunk grid with the tails of the full units handed to the CTAs
    of the diagonal units: full coverage, one main piece per CTA starting at its chunk's first k-step (so the
    CTAs of a chunk walk the same k window), balanced weights; not applicable shapes return no table."""
    table = _syrk_table(tiles, rows, ctas, -19)
    assert table is not None
    utab, cfirst, tfirst, clist = table
    n_tiles = tiles * (tiles + 1) // 2
    S = ctas // n_tiles
    ks = -(-rows // 16)
    starts = {16 * (ks * sc // S) for sc in range(S)}
    for b in range(n_tiles * S):
        first = utab[clist[cfirst[b]]]
        assert first[1] in starts, (b, first)
    loads = _check_syrk_table(tiles, rows, ctas, table, 10 ** 9)
    busy = [w for w in loads if w]
    mean = sum(busy) / len(busy)
    assert len(busy) == ctas  # the CTAs without a unit of their own take tails too
    assert max(busy) <= 1.01 * mean and min(busy) >= 0.98 * mean, (max(busy), mean, min(busy))
    assert _syrk_table(32, 65536, 148, -19) is None and _syrk_table(1, 40000, 148, -19) is None
    assert _syrk_table(2, 32768, 148, -19) is None  # chunks too short
