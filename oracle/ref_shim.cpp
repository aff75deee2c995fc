// ref_shim.cpp — extern "C" adapter over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. oracle/Makefile compiles the reference sources in
// place (/root/reference/proj/src/*.cpp, namespace renamed svdkit -> svdkit_ref
// with -Dsvdkit=svdkit_ref) together with this file into
// oracle/_ref/libsvdkit_ref.so. Tests use it to pin the C restatement
// (svdk_oracle.c) and to generate golden vectors; bench.py --impl reference
// uses it as the reference CPU arm. No reference source is copied here.
//
// Signatures mirror svdk_oracle.h (same buffers, same status codes) with a
// ref_ prefix.
#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "svdkit/dense_matrix.hpp"
#include "svdkit/errors.hpp"
#include "svdkit/kernels.hpp"
#include "svdkit/pca.hpp"
#include "svdkit/svd_methods.hpp"

namespace R = svdkit;  // expands to svdkit_ref under -Dsvdkit=svdkit_ref

namespace {

thread_local double g_residual = 0.0;

R::DenseMatrix wrap(const double* p, std::size_t r, std::size_t c) {
    return R::DenseMatrix(r, c, std::vector<double>(p, p + r * c));
}

void put(const R::DenseMatrix& m, double* out) {
    if (!m.data().empty()) std::memcpy(out, m.data().data(), m.data().size() * sizeof(double));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const R::DimensionError&) {
        return 1;
    } catch (const R::ParamError&) {
        return 2;
    } catch (const R::NumericalError& e) {
        g_residual = e.residual();
        return 3;
    } catch (...) {
        return 9;
    }
}

void put_svd(const R::SvdResult& s, double* u, double* sigma, double* v, std::size_t* rank) {
    put(s.u, u);
    if (!s.sigma.empty()) std::memcpy(sigma, s.sigma.data(), s.sigma.size() * sizeof(double));
    put(s.v, v);
    *rank = s.rank;
}

}  // namespace

extern "C" {

double ref_last_residual() { return g_residual; }

int ref_gaussian_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed, double* out) {
    return guard([&] { put(R::gaussian_matrix(rows, cols, R::RngSeed{seed}), out); });
}

int ref_matmul(const double* a, std::size_t m, std::size_t n, const double* b, std::size_t l,
               double* c) {
    return guard([&] { put(R::matmul(wrap(a, m, n), wrap(b, n, l)), c); });
}

int ref_matmul_tl(const double* a, std::size_t m, std::size_t n, const double* b, std::size_t l,
                  double* c) {
    return guard([&] { put(R::matmul_transposed_left(wrap(a, m, n), wrap(b, m, l)), c); });
}

int ref_gram(const double* a, std::size_t m, std::size_t n, double* g) {
    return guard([&] { put(R::gram(wrap(a, m, n)), g); });
}

double ref_frobenius_norm_sq(const double* a, std::size_t m, std::size_t n) {
    return R::frobenius_norm_sq(wrap(a, m, n));
}

int ref_qr_thin(const double* h, std::size_t m, std::size_t p, double* q, double* r,
                std::size_t* rank) {
    return guard([&] {
        R::QrResult res = R::qr_thin(wrap(h, m, p));
        put(res.q, q);
        if (r) put(res.r, r);
        if (rank) *rank = res.rank;
    });
}

int ref_eig_sym(const double* s, std::size_t n, int max_sweeps, double* w, double* v) {
    return guard([&] {
        R::EigResult e = R::eig_sym(wrap(s, n, n), max_sweeps);
        std::memcpy(w, e.eigenvalues.data(), n * sizeof(double));
        put(e.eigenvectors, v);
    });
}

int ref_truncated_svd(const double* a, std::size_t m, std::size_t n, double* u, double* sigma,
                      double* v, std::size_t* rank) {
    return guard([&] { put_svd(R::truncated_svd(wrap(a, m, n)), u, sigma, v, rank); });
}

int ref_randomized_pca(const double* a, std::size_t m, std::size_t n, std::size_t l,
                       std::size_t q, std::uint64_t seed, double* u, double* sigma, double* v,
                       std::size_t* rank) {
    return guard([&] {
        R::MethodParams p{l, q, R::RngSeed{seed}};
        put_svd(R::randomized_pca(wrap(a, m, n), p), u, sigma, v, rank);
    });
}

int ref_krylov_svd(const double* a, std::size_t m, std::size_t n, std::size_t l, std::size_t i,
                   std::uint64_t seed, double* u, double* sigma, double* v, std::size_t* rank) {
    return guard([&] {
        R::MethodParams p{l, i, R::RngSeed{seed}};
        put_svd(R::krylov_svd(wrap(a, m, n), p), u, sigma, v, rank);
    });
}

int ref_center(const double* a, std::size_t m, std::size_t n, int orientation, double* centered,
               double* mean) {
    return guard([&] {
        R::CenterResult c = R::center(wrap(a, m, n), orientation == 0
                                                         ? R::Orientation::ColumnsAreExamples
                                                         : R::Orientation::RowsAreExamples);
        put(c.centered, centered);
        std::memcpy(mean, c.mean.data(), c.mean.size() * sizeof(double));
    });
}

int ref_select_components(const double* w, std::size_t count, double total, double threshold,
                          std::size_t* k) {
    return guard([&] {
        std::vector<double> ev(w, w + count);
        std::optional<std::size_t> r = R::select_components(ev, total, threshold);
        *k = r ? *r : 0;
    });
}

// fit_pca(RowsAreExamples | ColumnsAreExamples, method 0/1/2) -> basis, eigenvalues, total.
int ref_fit_pca(const double* a, std::size_t m, std::size_t n, int orientation, int method,
                std::size_t l, std::size_t q, std::uint64_t seed, int center, double* basis,
                double* eigenvalues, double* total, std::size_t* rank, double* mean) {
    return guard([&] {
        R::MethodParams p{l, q, R::RngSeed{seed}};
        R::PcaModel mdl = R::fit_pca(
            wrap(a, m, n),
            orientation == 0 ? R::Orientation::ColumnsAreExamples : R::Orientation::RowsAreExamples,
            method == 0 ? R::SvdMethod::Truncated
                        : (method == 1 ? R::SvdMethod::Randomized : R::SvdMethod::Krylov),
            p, center != 0);
        put(mdl.basis, basis);
        std::memcpy(eigenvalues, mdl.eigenvalues.data(), mdl.eigenvalues.size() * sizeof(double));
        *total = mdl.total_variance;
        *rank = mdl.eigenvalues.size();
        if (mean) std::memcpy(mean, mdl.mean.data(), mdl.mean.size() * sizeof(double));
    });
}

// residual_delta (pca.cpp:133-168), used by tests as the paper's accuracy metric.
int ref_residual_delta(const double* a, std::size_t m, std::size_t n, const double* u,
                       const double* sigma, const double* v, std::size_t rank, double* delta) {
    return guard([&] {
        R::SvdResult s;
        s.u = wrap(u, m, rank);
        s.v = wrap(v, n, rank);
        s.sigma.assign(sigma, sigma + rank);
        s.rank = rank;
        *delta = R::residual_delta(wrap(a, m, n), s);
    });
}

}  // extern "C"
