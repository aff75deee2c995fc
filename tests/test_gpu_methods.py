"""GPU parity of the SVD methods and the PCA pipeline against the compiled
reference (golden fixtures + live oracle at small sizes).

Bars (BASELINE.json north_star): eigenvalues within 1e-10 relative, principal-
angle sine <= 1e-8 (top-K subspace; per vector where the relative gap allows,
clusters compared as subspaces — SURVEY §8c), K exact.
"""
import os

import numpy as np
import pytest

from paper_1906_12085_b200 import errors
from tests.datagen import config_matrix
from tests.parity import eig_rel_err, orthogonality, per_vector_sines, subspace_sine

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"missing {name}")
    return np.load(p)


def check_svd(s, sigma_ref, v_ref, k=None, vtol=1e-8, etol=1e-10):
    assert s.rank == len(sigma_ref)
    assert eig_rel_err(s.sigma ** 2, sigma_ref ** 2) <= etol
    kk = k or len(sigma_ref)
    assert subspace_sine(s.v[:, :kk], v_ref[:, :kk]) <= vtol
    single, cluster = per_vector_sines(s.v[:, :v_ref.shape[1]], sigma_ref ** 2, v_ref)
    assert single <= vtol and cluster <= vtol
    assert orthogonality(s.v) <= 1e-10 and orthogonality(s.u) <= 1e-8


def test_truncated_kat(sk):
    s = sk.truncated_svd(np.array([[3.0, 0], [0, 4], [0, 0]]))
    assert s.sigma.tolist() == [4.0, 3.0]
    assert s.u.tolist() == [[0, 1], [1, 0], [0, 0]] and s.v.tolist() == [[0, 1], [1, 0]]


def test_zero_matrix_rank0(sk):
    assert sk.truncated_svd(np.zeros((5, 3))).rank == 0
    assert sk.randomized_pca(np.zeros((5, 3)), sk.MethodParams(2, 1, sk.RngSeed(7))).rank == 0


def test_method_errors(sk):
    with pytest.raises(errors.DimensionError):
        sk.truncated_svd(np.ones((2, 3)))
    with pytest.raises(errors.ParamError):
        sk.randomized_pca(np.ones((4, 3)), sk.MethodParams(4, 1))
    with pytest.raises(errors.ParamError):
        sk.krylov_svd(np.ones((4, 3)), sk.MethodParams(2, 2))
    with pytest.raises(errors.ParamError):
        sk.krylov_svd(np.ones((8, 3)), sk.MethodParams(2, 0))


def test_small_golden_all_methods(sk):
    gz = golden("small.npz")
    a = gz["a"]
    t = sk.truncated_svd(a)
    check_svd(t, gz["trunc_sigma"], gz["trunc_v"])
    # signs follow the reference convention (normalize_signs), so vectors compare directly
    assert np.max(np.abs(t.v - gz["trunc_v"])) < 1e-9
    r = sk.randomized_pca(a, sk.MethodParams(int(gz["l"]), int(gz["q"]), sk.RngSeed(int(gz["rseed"]))))
    check_svd(r, gz["rand_sigma"], gz["rand_v"])
    k = sk.krylov_svd(a, sk.MethodParams(int(gz["kl"]), int(gz["ki"]), sk.RngSeed(int(gz["rseed"]))))
    check_svd(k, gz["kry_sigma"], gz["kry_v"])
    lz = sk.lanczos_svd(a, 0, sk.RngSeed(5))
    check_svd(lz, gz["trunc_sigma"], gz["trunc_v"])


@pytest.mark.parametrize("method", ["truncated", "randomized", "krylov", "lanczos"])
def test_c1_fit_pca_vs_reference(sk, method):
    """BASELINE config 1 (20000 x 256, t = 0.95) through fit_pca + select_components."""
    gz = golden("c1.npz")
    a = config_matrix("c1", seed=int(gz["seed"]))
    key = "truncated" if method == "lanczos" else method
    l, q, rs = (int(x) for x in gz[f"{key}_params"])
    enum = {"truncated": sk.SvdMethod.Truncated, "randomized": sk.SvdMethod.Randomized,
            "krylov": sk.SvdMethod.Krylov, "lanczos": sk.SvdMethod.Lanczos}[method]
    params = sk.MethodParams(l if method != "lanczos" else 0, q, sk.RngSeed(rs))
    model = sk.fit_pca(a, sk.Orientation.RowsAreExamples, enum, params, True)
    lam_ref, v_ref = gz[f"{key}_lambda"], gz[f"{key}_v"]
    assert abs(model.total_variance - float(gz["total"])) <= 1e-12 * float(gz["total"])
    assert eig_rel_err(model.eigenvalues, lam_ref) <= 1e-10
    k_ref = int(gz[f"{key}_k"])
    k = sk.select_components(model.eigenvalues, model.total_variance, float(gz["threshold"]))
    assert k == k_ref == 214
    assert subspace_sine(model.basis[:, :k], v_ref[:, :k]) <= 1e-8
    single, cluster = per_vector_sines(model.basis, lam_ref, v_ref)
    assert single <= 1e-8 and cluster <= 1e-8


@pytest.mark.parametrize("method", ["truncated", "randomized"])
def test_fit_pca_streamed_upload(sk, monkeypatch, method):
    """Host-buffer fit_pca with the upload streamed under the first pass
    (stream_fit.cu) on c1: truncated in two column chunks (192 + 64 columns),
    randomized in 7 row chunks (each centred by its own means, closed-form
    correction to the global mean); same golden bars as the plain path; then a matrix with large
    column means (|mu| ~ 1e3 x the spread) against the plain path."""
    gz = golden("c1.npz")
    a = config_matrix("c1", seed=int(gz["seed"]))
    l, q, rs = (int(x) for x in gz[f"{method}_params"])
    enum = sk.SvdMethod.Truncated if method == "truncated" else sk.SvdMethod.Randomized
    params = sk.MethodParams(l, q, sk.RngSeed(rs))
    monkeypatch.setenv("SVDK_STREAM_COLS", "192")  # truncated: column chunks
    monkeypatch.setenv("SVDK_STREAM_ROWS", "3000")  # randomized: row chunks (7, last partial)
    model = sk.fit_pca(a, sk.Orientation.RowsAreExamples, enum, params, True)
    lam_ref, v_ref = gz[f"{method}_lambda"], gz[f"{method}_v"]
    assert abs(model.total_variance - float(gz["total"])) <= 1e-12 * float(gz["total"])
    assert eig_rel_err(model.eigenvalues, lam_ref) <= 1e-10
    k = sk.select_components(model.eigenvalues, model.total_variance, float(gz["threshold"]))
    assert k == int(gz[f"{method}_k"]) == 214
    assert subspace_sine(model.basis[:, :k], v_ref[:, :k]) <= 1e-8
    single, cluster = per_vector_sines(model.basis, lam_ref, v_ref)
    assert single <= 1e-8 and cluster <= 1e-8
    # large, chunk-varying column means
    rng = np.random.default_rng(5)
    spread = float(np.sqrt(gz["total"] / a.size))
    shifted = np.asfortranarray(a + 1e3 * spread * (1.0 + rng.standard_normal(256))[None, :]
                                + spread * np.linspace(0.0, 5.0, 20000)[:, None])
    streamed = sk.fit_pca(shifted, sk.Orientation.RowsAreExamples, enum, params, True)
    monkeypatch.setenv("SVDK_STREAM", "0")
    plain = sk.fit_pca(shifted, sk.Orientation.RowsAreExamples, enum, params, True)
    assert np.max(np.abs(streamed.mean - plain.mean)) <= 1e-12 * np.max(np.abs(plain.mean))
    assert abs(streamed.total_variance - plain.total_variance) <= 1e-11 * plain.total_variance
    assert eig_rel_err(streamed.eigenvalues, plain.eigenvalues) <= 1e-10
    kk = sk.select_components(plain.eigenvalues, plain.total_variance, 0.95)
    assert subspace_sine(streamed.basis[:, :kk], plain.basis[:, :kk]) <= 1e-8


def test_live_oracle_random_shapes(sk, ref):
    rng = np.random.default_rng(21)
    for m, n in ((40, 40), (333, 65), (1000, 129)):
        a = np.asfortranarray(rng.standard_normal((m, n)))
        s, r = sk.truncated_svd(a), ref.truncated_svd(a)
        check_svd(s, r.sigma, r.v)
        rp = sk.randomized_pca(a, sk.MethodParams(n, 2, sk.RngSeed(3)))
        rr = ref.randomized_pca(a, n, 2, 3)
        check_svd(rp, rr.sigma, rr.v, vtol=1e-7)


def test_compute_svd_any_wide(sk, ref):
    a = np.asfortranarray(np.random.default_rng(8).standard_normal((30, 90)))
    s = sk.compute_svd_any(a, sk.SvdMethod.Truncated, sk.MethodParams(1, 1))
    r = ref.truncated_svd(np.asfortranarray(a.T))
    assert s.u.shape == (30, 30) and s.v.shape == (90, 30)
    assert eig_rel_err(s.sigma, r.sigma) < 1e-12
    assert np.linalg.norm(a - (s.u * s.sigma) @ s.v.T) < 1e-12 * np.linalg.norm(a)


def test_fit_pca_columns_are_examples(sk, ref):
    a = np.asfortranarray(np.random.default_rng(10).standard_normal((40, 300)))
    model = sk.fit_pca(a, sk.Orientation.ColumnsAreExamples, sk.SvdMethod.Truncated, sk.MethodParams(), True)
    c, mean = ref.center(a, 0)
    r = ref.truncated_svd(np.asfortranarray(c.T))  # wide -> factor the transpose; basis = U of c = V of c^T
    assert model.basis.shape[0] == 40 and np.allclose(model.mean, mean, atol=1e-14)
    assert eig_rel_err(model.eigenvalues, r.sigma ** 2) < 1e-10


def test_residual_delta_transform_truncate(sk, ref):
    a = np.asfortranarray(np.random.default_rng(14).standard_normal((500, 30)))
    s = sk.truncated_svd(a)
    d = sk.residual_delta(a, s)
    d_ref = ref.residual_delta(a, s.u, s.sigma, s.v)
    assert d < 1e-13 and abs(d - d_ref) < 1e-13
    s5 = sk.truncate_rank(s, 5)
    d5, d5_ref = sk.residual_delta(a, s5), ref.residual_delta(a, s5.u, s5.sigma, s5.v)
    assert abs(d5 - d5_ref) <= 1e-12 * d5_ref  # Eckart-Young residual of the rank-5 truncation
    with pytest.raises(errors.ParamError):
        sk.truncate_rank(s, 0)
    with pytest.raises(errors.ParamError):
        sk.residual_delta(np.zeros((4, 2)), sk.SvdResult(np.zeros((4, 1)), np.ones(1), np.zeros((2, 1)), 1))
    model = sk.fit_pca(a, sk.Orientation.RowsAreExamples, sk.SvdMethod.Truncated, sk.MethodParams(), True)
    c = sk.center(a, sk.Orientation.RowsAreExamples).centered
    y = sk.transform(model, c)
    assert np.allclose(y, c @ model.basis, rtol=0, atol=1e-12)


@pytest.mark.parametrize("gemv", ["cluster:1", "cluster:2", "cluster:4", "cluster:8", "twopass:4"])
def test_lanczos_gemv_forms_ragged(sk, ref, monkeypatch, gemv):
    """Every GEMV-pair form (cluster size 1/2/4/8, two-pass fallback) on shapes
    with partial 64-row slabs, partial 32-column tiles, m < 64 and CTAs that own
    no columns (n < cluster x 32) — all against the reference truncated_svd."""
    mode, cs = gemv.split(":")
    monkeypatch.setenv("SVDK_GEMV", mode)
    monkeypatch.setenv("SVDK_GEMV_CS", cs)
    rng = np.random.default_rng(31)
    for m, n in ((50, 7), (63, 40), (1000, 130), (4099, 257)):
        a = np.asfortranarray(rng.standard_normal((m, n)))
        r = ref.truncated_svd(a)
        s = sk.lanczos_svd(a, 0, sk.RngSeed(2))
        check_svd(s, r.sigma, r.v)


def test_lanczos_breakdown_restart(sk, ref):
    """Rank-deficient A: the Krylov space is invariant after rank(A) steps, the
    device-side breakdown test fires and every later step restarts inside the
    numerical null space. The true spectrum and subspace must match the
    reference; the remaining Ritz values sit at the rounding floor (the
    reference's own rank cut also keeps such noise: its Gram eigenvalues are
    +-1e-16 ||A||^2, so sigma ~ 1e-8 sigma_1 passes the 1e-12 cut)."""
    rng = np.random.default_rng(12)
    for rank, (m, n) in ((5, (400, 40)), (17, (3000, 96))):
        a = np.asfortranarray(rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n)))
        r = ref.truncated_svd(a)
        s = sk.lanczos_svd(a, 0, sk.RngSeed(9))
        assert r.rank >= rank and s.rank >= rank
        assert eig_rel_err(s.sigma[:rank] ** 2, r.sigma[:rank] ** 2) <= 1e-10
        assert np.all(s.sigma[rank:] <= 1e-6 * s.sigma[0])
        assert subspace_sine(s.v[:, :rank], r.v[:, :rank]) <= 1e-8
        assert orthogonality(s.v) <= 1e-10 and orthogonality(s.u[:, :rank]) <= 1e-8


def test_lanczos_tridiagonal_solver_matches_dense(sk, monkeypatch):
    """The O(k^2) tridiagonal eigensolver (bisection + twisted factorisation +
    CholeskyQR certification, tridiag.cu) against the dense Jacobi solve of
    the same Lanczos T (SVDK_LANCZOS_TRIDIAG=0), on c2's spectrum."""
    from tests.datagen import make_matrix
    a = make_matrix(6000, 512, "c2", seed=5)
    fast = sk.lanczos_svd(a, 0, sk.RngSeed(3))
    monkeypatch.setenv("SVDK_LANCZOS_TRIDIAG", "0")
    dense = sk.lanczos_svd(a, 0, sk.RngSeed(3))
    assert fast.rank == dense.rank
    assert eig_rel_err(fast.sigma ** 2, dense.sigma ** 2) <= 1e-12
    single, cluster = per_vector_sines(fast.v, dense.sigma ** 2, dense.v)
    assert single <= 1e-9 and cluster <= 1e-9
    assert orthogonality(fast.v) <= 1e-12
