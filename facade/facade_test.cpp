// facade_test.cpp — a reference-style caller compiled against the drop-in
// headers (include/svdkit/*.hpp) and linked to libsvdkit.so. It uses only the
// reference API; run on a GPU box by tests/test_gpu_facade.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "svdkit/kernels.hpp"
#include "svdkit/pca.hpp"
#include "svdkit/svd_methods.hpp"

using namespace svdkit;

static int failures = 0;
#define EXPECT(cond)                                                  \
    do {                                                              \
        if (!(cond)) {                                                \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                               \
        }                                                             \
    } while (0)

int main() {
    // kernels (SPEC.md examples / SURVEY 4 known answers)
    DenseMatrix c = matmul(DenseMatrix::from_rows({{1, 2}, {3, 4}}), DenseMatrix::from_rows({{5, 6}, {7, 8}}));
    EXPECT(c(0, 0) == 19 && c(0, 1) == 22 && c(1, 0) == 43 && c(1, 1) == 50);
    try {
        matmul(DenseMatrix(2, 3), DenseMatrix(2, 3));
        EXPECT(false);
    } catch (const DimensionError&) {
    }
    QrResult qr = qr_thin(DenseMatrix::from_rows({{3}, {4}}));
    EXPECT(std::fabs(qr.q(0, 0) - 0.6) < 1e-15 && std::fabs(qr.r(0, 0) - 5) < 1e-14 && qr.rank == 1);
    EigResult e = eig_sym(DenseMatrix::from_rows({{2, 1}, {1, 2}}));
    EXPECT(std::fabs(e.eigenvalues[0] - 3) < 1e-14 && std::fabs(e.eigenvalues[1] - 1) < 1e-14);
    try {
        eig_sym(DenseMatrix::from_rows({{1, 0.5}, {0, 1}}));
        EXPECT(false);
    } catch (const ParamError&) {
    }
    DenseMatrix g = gaussian_matrix(3, 2, RngSeed{42});
    EXPECT(g.data()[0] == -0.48121769980184492 && g.data()[5] == 0.25135417655083486);

    // methods
    SvdResult s = truncated_svd(DenseMatrix::from_rows({{3, 0}, {0, 4}, {0, 0}}));
    EXPECT(s.rank == 2 && s.sigma[0] == 4.0 && s.sigma[1] == 3.0);
    EXPECT(s.u(1, 0) == 1.0 && s.v(1, 0) == 1.0 && s.u(0, 1) == 1.0 && s.v(0, 1) == 1.0);
    EXPECT(truncated_svd(DenseMatrix(5, 3)).rank == 0);
    try {
        truncated_svd(DenseMatrix(2, 3));
        EXPECT(false);
    } catch (const DimensionError&) {
    }
    try {
        randomized_pca(DenseMatrix(4, 3), MethodParams{4, 1, RngSeed{0}});
        EXPECT(false);
    } catch (const ParamError&) {
    }

    // a random tall matrix through every method agrees on the spectrum
    const std::size_t m = 400, n = 24;
    DenseMatrix a = gaussian_matrix(m, n, RngSeed{7});
    SvdResult t = truncated_svd(a);
    SvdResult r = randomized_pca(a, MethodParams{n, 2, RngSeed{3}});
    SvdResult k = krylov_svd(a, MethodParams{8, 2, RngSeed{3}});
    SvdResult l = lanczos_svd(a, MethodParams{0, 0, RngSeed{3}});
    EXPECT(t.rank == n && r.rank == n && k.rank == n && l.rank == n);
    for (std::size_t i = 0; i < n; ++i) {
        EXPECT(std::fabs(r.sigma[i] - t.sigma[i]) <= 1e-10 * t.sigma[i]);
        EXPECT(std::fabs(k.sigma[i] - t.sigma[i]) <= 1e-10 * t.sigma[i]);
        EXPECT(std::fabs(l.sigma[i] - t.sigma[i]) <= 1e-10 * t.sigma[i]);
    }
    EXPECT(residual_delta(a, t) < 1e-12);
    SvdResult t3 = truncate_rank(t, 3);
    EXPECT(t3.rank == 3 && t3.u.cols() == 3 && t3.sigma.size() == 3);
    EXPECT(method_from_name("lanczos") == SvdMethod::Lanczos && !method_from_name("qr"));

    // PCA
    PcaModel model = fit_pca(a, Orientation::RowsAreExamples, SvdMethod::Truncated, MethodParams{}, true);
    auto kk = select_components(model.eigenvalues, model.total_variance, 0.9);
    EXPECT(kk.has_value() && *kk >= 1 && *kk <= n);
    EXPECT(std::fabs(model.total_variance - total_variance(center(a, Orientation::RowsAreExamples).centered)) <=
           1e-10 * model.total_variance);
    DenseMatrix y = transform(model, center(a, Orientation::RowsAreExamples).centered);
    EXPECT(y.rows() == m && y.cols() == model.basis.cols());
    EXPECT(select_components({4, 3, 2, 1}, 10, 0.7) == 2);
    EXPECT(!select_components({4, 3, 2, 1}, 11, 1.0).has_value());

    std::printf("facade_test: %s (%d failures)\n", failures ? "FAILED" : "ok", failures);
    return failures ? 1 : 0;
}
