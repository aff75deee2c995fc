"""GPU parts of the host-tool rows: IDX expansion kernel
bit-exact against the reference images_to_matrix, and the benchmark grid
running its factorisations on the engine."""
import io

import numpy as np
import pytest

from tests.conftest import HAS_GPU
from tests.test_host_tools import idx_bytes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rt():
    from oracle.pyoracle import RefTools, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built")
    return RefTools()


@pytest.mark.parametrize("dims", [(1, 1, 1), (3, 28, 28), (70, 9, 11), (129, 28, 28), (1000, 3, 50)])
def test_images_to_matrix_bit_exact(rt, dims):
    if not HAS_GPU:
        pytest.skip("no GPU")
    from paper_1906_12085_b200 import idx_io
    data = idx_bytes(*dims)
    got = idx_io.images_to_matrix(idx_io.parse_idx_images(data))
    want = rt.images_to_matrix(data)
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_images_to_matrix_dev_strided():
    if not HAS_GPU:
        pytest.skip("no GPU")
    import torch
    from paper_1906_12085_b200 import _lib, idx_io
    count, p, ldo = 300, 784, 304
    rng = np.random.default_rng(4)
    px = rng.integers(0, 256, count * p, dtype=np.uint8)
    d_px = torch.from_numpy(px).cuda()
    out = torch.full((p, ldo), -1.0, dtype=torch.float64, device="cuda")  # column-major view: out.T
    ctx = _lib.default_context()
    torch.cuda.synchronize()
    idx_io.images_to_matrix_dev(ctx, d_px.data_ptr(), count, p, out.data_ptr(), ldo)
    ctx.sync()
    got = out.cpu().numpy()  # row j = column j of the count x p matrix
    want = px.reshape(count, p).astype(np.float64) / 255.0
    assert np.array_equal(got[:, :count].T, want)
    assert (got[:, count:] == -1.0).all()  # padding rows untouched


def test_run_grid_on_gpu(rt):
    if not HAS_GPU:
        pytest.skip("no GPU")
    from paper_1906_12085_b200 import bench_grid
    from paper_1906_12085_b200.svdkit import RngSeed, SvdMethod
    cfg = bench_grid.BenchConfig([400, 200], [40, 64], [SvdMethod.Truncated, SvdMethod.Randomized,
                                                        SvdMethod.Krylov, SvdMethod.Truncated],
                                 repeats=2, seed=RngSeed(7), l_fraction=0.5, iterations=1,
                                 memory_cap_bytes=8.0 * 400 * 40 + 1)
    res = bench_grid.run_grid(cfg)
    # 400x64 exceeds the memory cap for every method; nothing else is skipped
    assert sorted((s.m, s.n) for s in res.skipped) == [(400, 64)] * 3
    assert all("cap is" in s.reason for s in res.skipped)
    cells = [(r.m, r.n, r.method) for r in res.records]
    assert cells == [(m, n, meth) for m, n in [(200, 40), (200, 64), (400, 40)]
                     for meth in (SvdMethod.Krylov, SvdMethod.Randomized, SvdMethod.Truncated)]
    for r in res.records:
        assert r.repeats == 2 and r.mean_seconds > 0 and r.std_seconds >= 0
        l = bench_grid.sketch_width_for(cfg, r.n)
        want = {SvdMethod.Truncated: rt.cost(0, r.m, r.n), SvdMethod.Randomized: rt.cost(1, r.m, r.n, l, 1),
                SvdMethod.Krylov: rt.cost(3, r.m, r.n, l, 1)}[r.method]
        assert (r.model_flops, r.model_space_bytes) == (want[0], want[2])
        if r.method == SvdMethod.Truncated:
            assert r.delta < 1e-12  # exact factorisation
        else:
            assert 0.0 < r.delta < 1.0  # rank-l approximation of a Gaussian matrix
    text = bench_grid.to_csv(res.records)
    assert text.splitlines()[0] == bench_grid.CSV_HEADER.strip()
    assert len(text.splitlines()) == 1 + len(res.records)
    rep = bench_grid.format_report(bench_grid.summarize_ordering(res.records))
    assert rep.startswith("cell") and "ranking agreement:" in rep
    # CLI end to end
    out = io.StringIO()
    import contextlib
    with contextlib.redirect_stdout(out):
        assert bench_grid.main(["--rows", "200", "--cols", "40", "--methods", "truncated,randomized",
                                "--repeats", "1", "--report"]) == 0
    assert out.getvalue().startswith(bench_grid.CSV_HEADER)
