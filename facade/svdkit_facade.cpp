// svdkit_facade.cpp — the reference's C++ API (include/svdkit/svdkit.hpp)
// implemented over the B200 engine's C-ABI (include/svdk.h).
//
// Callers keep their code: DenseMatrix in, DenseMatrix / result structs out,
// reference exception types on error. Host-side work here is limited to
// argument validation, buffer marshalling and pure data movement
// (truncate_rank, wide/tall swaps); every arithmetic kernel runs on the GPU
// through libsvdk.so. One engine context per host thread (lazy, device from
// SVDK_DEVICE, default 0), matching the reference's "pure functions, callers
// may parallelise across independent calls" model.
#include <cmath>
#include <cstdlib>
#include <memory>

#include "svdk.h"
#include "svdkit/svdkit.hpp"

namespace svdkit {

namespace {

struct CtxHolder {
    svdk_ctx* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) svdk_ctx_destroy(ctx);
    }
};

[[noreturn]] void rethrow(int code, std::size_t offset = 0) {
    const std::string msg = svdk_last_error();
    switch (code) {
        case SVDK_E_FORMAT:
            throw FormatError(msg, offset);
        case SVDK_E_IO:
            throw IoError(msg);
        case SVDK_E_DIM:
            throw DimensionError(msg);
        case SVDK_E_PARAM:
            throw ParamError(msg);
        case SVDK_E_NUMERICAL:
            throw NumericalError(msg, svdk_last_residual());
        default:
            throw EngineError("svdk engine: " + msg);
    }
}

void check(int code, std::size_t offset = 0) {
    if (code != SVDK_OK) rethrow(code, offset);
}

svdk_ctx* ctx() {
    thread_local CtxHolder holder;
    if (!holder.ctx) {
        const char* dev = std::getenv("SVDK_DEVICE");
        check(svdk_ctx_create(dev ? std::atoi(dev) : 0, &holder.ctx));
    }
    return holder.ctx;
}

void check_finite(const std::vector<double>& v) {
    for (double x : v)
        if (!std::isfinite(x)) throw ParamError("DenseMatrix: non-finite entry (NaN/Inf) rejected");
}

int64_t I(std::size_t x) { return static_cast<int64_t>(x); }

// first r columns of a rows x cap column-major buffer
DenseMatrix take_cols(std::size_t rows, std::size_t r, const std::vector<double>& buf) {
    return DenseMatrix(rows, r, std::vector<double>(buf.begin(), buf.begin() + rows * r));
}

int method_id(SvdMethod m) {
    switch (m) {
        case SvdMethod::Truncated:
            return SVDK_TRUNCATED;
        case SvdMethod::Randomized:
            return SVDK_RANDOMIZED;
        case SvdMethod::Krylov:
            return SVDK_KRYLOV;
        case SvdMethod::Lanczos:
            return SVDK_LANCZOS;
    }
    throw ParamError("compute_svd: unknown method");
}

// Output width bound of a method on a tall m x n input.
std::size_t width_of(SvdMethod m, std::size_t n, const MethodParams& p) {
    switch (m) {
        case SvdMethod::Randomized:
            return std::max<std::size_t>(p.sketch_width, 1);
        case SvdMethod::Krylov:
            return std::max<std::size_t>(std::min((p.power_iterations + 1) * p.sketch_width, n), 1);
        case SvdMethod::Lanczos:
            return (p.sketch_width == 0 || p.sketch_width > n) ? n : p.sketch_width;
        default:
            return std::max<std::size_t>(n, 1);
    }
}

}  // namespace

// shared with svdkit_tools.cpp (facade-internal, not part of the API)
namespace detail {
svdk_ctx* engine_ctx() { return ctx(); }
void engine_check(int code, std::size_t offset) { check(code, offset); }
}  // namespace detail

// ---------------------------------------------------------------- DenseMatrix
DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols)
    : nr_(rows), nc_(cols), v_(rows * cols, 0.0) {}

DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols, std::vector<double> data)
    : nr_(rows), nc_(cols), v_(std::move(data)) {
    if (v_.size() != nr_ * nc_)
        throw ParamError("DenseMatrix: data length " + std::to_string(v_.size()) +
                         " does not match " + std::to_string(nr_) + "x" + std::to_string(nc_));
    check_finite(v_);
}

DenseMatrix DenseMatrix::identity(std::size_t n) {
    DenseMatrix m(n, n);
    for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
}

DenseMatrix DenseMatrix::from_rows(std::initializer_list<std::initializer_list<double>> rows) {
    const std::size_t r = rows.size(), c = r ? rows.begin()->size() : 0;
    DenseMatrix m(r, c);
    std::size_t i = 0;
    for (const auto& row : rows) {
        if (row.size() != c) throw ParamError("DenseMatrix::from_rows: ragged rows");
        std::size_t j = 0;
        for (double x : row) {
            if (!std::isfinite(x)) throw ParamError("DenseMatrix: non-finite entry (NaN/Inf) rejected");
            m(i, j++) = x;
        }
        ++i;
    }
    return m;
}

std::string shape_string(const DenseMatrix& a) {
    return std::to_string(a.rows()) + "x" + std::to_string(a.cols());
}

// ---------------------------------------------------------------- kernels
DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.cols() != b.rows())
        throw DimensionError("matmul: inner dimensions differ, a is " + shape_string(a) + ", b is " +
                             shape_string(b));
    std::vector<double> c(a.rows() * b.cols());
    check(svdk_matmul(ctx(), a.data().data(), I(a.rows()), I(a.cols()), b.data().data(), I(b.cols()),
                      c.data()));
    return DenseMatrix(a.rows(), b.cols(), std::move(c));
}

DenseMatrix matmul_transposed_left(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.rows() != b.rows())
        throw DimensionError("matmul_transposed_left: row counts differ, a is " + shape_string(a) +
                             ", b is " + shape_string(b));
    std::vector<double> c(a.cols() * b.cols());
    check(svdk_matmul_transposed_left(ctx(), a.data().data(), I(a.rows()), I(a.cols()),
                                      b.data().data(), I(b.cols()), c.data()));
    return DenseMatrix(a.cols(), b.cols(), std::move(c));
}

DenseMatrix transpose(const DenseMatrix& a) {
    std::vector<double> t(a.size());
    if (!a.empty()) check(svdk_transpose(ctx(), a.data().data(), I(a.rows()), I(a.cols()), t.data()));
    return DenseMatrix(a.cols(), a.rows(), std::move(t));
}

DenseMatrix gram(const DenseMatrix& a) {
    std::vector<double> g(a.cols() * a.cols());
    if (a.cols()) check(svdk_gram(ctx(), a.data().data(), I(a.rows()), I(a.cols()), g.data()));
    return DenseMatrix(a.cols(), a.cols(), std::move(g));
}

double frobenius_norm_sq(const DenseMatrix& a) {
    if (a.empty()) return 0.0;
    double out = 0.0;
    check(svdk_frobenius_norm_sq(ctx(), a.data().data(), I(a.rows()), I(a.cols()), &out));
    return out;
}

double frobenius_norm(const DenseMatrix& a) { return std::sqrt(frobenius_norm_sq(a)); }

QrResult qr_thin(const DenseMatrix& h) {
    if (h.rows() < h.cols())
        throw DimensionError("qr_thin: need rows >= cols, got " + shape_string(h));
    std::vector<double> q(h.size()), r(h.cols() * h.cols());
    int64_t rank = 0;
    if (h.cols())
        check(svdk_qr_thin(ctx(), h.data().data(), I(h.rows()), I(h.cols()), q.data(), r.data(), &rank));
    return QrResult{DenseMatrix(h.rows(), h.cols(), std::move(q)),
                    DenseMatrix(h.cols(), h.cols(), std::move(r)), static_cast<std::size_t>(rank)};
}

EigResult eig_sym(const DenseMatrix& s) { return eig_sym(s, 30); }

EigResult eig_sym(const DenseMatrix& s, int max_sweeps) {
    if (s.rows() != s.cols())
        throw DimensionError("eig_sym: matrix not square, got " + shape_string(s));
    const std::size_t n = s.rows();
    EigResult out;
    out.eigenvalues.resize(n);
    std::vector<double> v(n * n);
    if (n) check(svdk_eig_sym(ctx(), s.data().data(), I(n), max_sweeps, out.eigenvalues.data(), v.data()));
    out.eigenvectors = DenseMatrix(n, n, std::move(v));
    return out;
}

DenseMatrix gaussian_matrix(std::size_t rows, std::size_t cols, RngSeed seed) {
    if (rows < 1 || cols < 1) throw ParamError("gaussian_matrix: rows and cols must be >= 1");
    std::vector<double> g(rows * cols);
    check(svdk_gaussian_matrix(I(rows), I(cols), seed.value, g.data()));
    return DenseMatrix(rows, cols, std::move(g));
}

// ---------------------------------------------------------------- methods
const char* method_name(SvdMethod method) {
    switch (method) {
        case SvdMethod::Truncated:
            return "truncated";
        case SvdMethod::Randomized:
            return "randomized";
        case SvdMethod::Krylov:
            return "krylov";
        case SvdMethod::Lanczos:
            return "lanczos";
    }
    return "unknown";
}

std::optional<SvdMethod> method_from_name(std::string_view name) {
    for (SvdMethod m : {SvdMethod::Truncated, SvdMethod::Randomized, SvdMethod::Krylov, SvdMethod::Lanczos})
        if (name == method_name(m)) return m;
    return std::nullopt;
}

MethodParams MethodParams::defaults_for(std::size_t n, RngSeed seed) {
    return MethodParams{(n + 1) / 2, 1, seed};
}

namespace {
SvdResult run(const DenseMatrix& a, SvdMethod method, const MethodParams& p) {
    const std::size_t m = a.rows(), n = a.cols();
    if (m < n)
        throw DimensionError(std::string(method_name(method)) + ": needs rows >= cols, got " +
                             shape_string(a));
    if (n == 0) throw DimensionError(std::string(method_name(method)) + ": empty input");
    const std::size_t w = width_of(method, n, p);
    std::vector<double> u(m * w), s(std::max(w, n)), v(n * w);
    int64_t rank = 0;
    check(svdk_compute_svd(ctx(), a.data().data(), I(m), I(n), method_id(method), I(p.sketch_width),
                           I(p.power_iterations), p.seed.value, u.data(), s.data(), v.data(), &rank));
    SvdResult out;
    out.rank = static_cast<std::size_t>(rank);
    out.u = take_cols(m, out.rank, u);
    out.v = take_cols(n, out.rank, v);
    out.sigma.assign(s.begin(), s.begin() + out.rank);
    out.method = method;
    return out;
}
}  // namespace

SvdResult truncated_svd(const DenseMatrix& a) { return run(a, SvdMethod::Truncated, MethodParams{}); }
SvdResult randomized_pca(const DenseMatrix& a, const MethodParams& p) {
    return run(a, SvdMethod::Randomized, p);
}
SvdResult krylov_svd(const DenseMatrix& a, const MethodParams& p) { return run(a, SvdMethod::Krylov, p); }
SvdResult lanczos_svd(const DenseMatrix& a, const MethodParams& p) { return run(a, SvdMethod::Lanczos, p); }

// svd_methods.cpp:198-225 — pure data movement
SvdResult truncate_rank(const SvdResult& s, std::size_t k) {
    if (k < 1 || k > s.rank)
        throw ParamError("truncate_rank: k = " + std::to_string(k) + " outside [1, rank = " +
                         std::to_string(s.rank) + "]");
    if (k == s.rank) return s;
    SvdResult out;
    out.u = take_cols(s.u.rows(), k, s.u.data());
    out.v = take_cols(s.v.rows(), k, s.v.data());
    out.sigma.assign(s.sigma.begin(), s.sigma.begin() + static_cast<std::ptrdiff_t>(k));
    out.rank = k;
    out.method = s.method;
    return out;
}

SvdResult compute_svd(const DenseMatrix& a, SvdMethod method, const MethodParams& p) {
    return run(a, method, p);
}

SvdResult compute_svd_any(const DenseMatrix& a, SvdMethod method, const MethodParams& p) {
    if (a.rows() >= a.cols()) return compute_svd(a, method, p);
    SvdResult s = compute_svd(transpose(a), method, p);
    std::swap(s.u, s.v);
    return s;
}

// ---------------------------------------------------------------- PCA
CenterResult center(const DenseMatrix& a, Orientation orientation) {
    const bool cols_ex = orientation == Orientation::ColumnsAreExamples;
    CenterResult out;
    out.mean.resize(cols_ex ? a.rows() : a.cols());
    std::vector<double> c(a.size());
    check(svdk_center(ctx(), a.data().data(), I(a.rows()), I(a.cols()),
                      cols_ex ? SVDK_COLUMNS_ARE_EXAMPLES : SVDK_ROWS_ARE_EXAMPLES, c.data(),
                      out.mean.data()));
    out.centered = DenseMatrix(a.rows(), a.cols(), std::move(c));
    return out;
}

double total_variance(const DenseMatrix& centered) { return frobenius_norm_sq(centered); }

std::optional<std::size_t> select_components(const std::vector<double>& eigenvalues, double total,
                                             double threshold) {
    int64_t k = 0;
    check(svdk_select_components(ctx(), eigenvalues.data(), I(eigenvalues.size()), total, threshold, &k));
    if (k == 0) return std::nullopt;
    return static_cast<std::size_t>(k);
}

PcaModel fit_pca(const DenseMatrix& data, Orientation orientation, SvdMethod method,
                 const MethodParams& params, bool center_data) {
    const bool cols_ex = orientation == Orientation::ColumnsAreExamples;
    const std::size_t m = data.rows(), n = data.cols(), tn = std::min(m, n);
    const std::size_t w = width_of(method, tn, params);
    const std::size_t basis_rows = cols_ex ? m : n;
    std::vector<double> basis(basis_rows * w), eig(w), mean(cols_ex ? m : n);
    double total = 0.0;
    int64_t rank = 0;
    check(svdk_fit_pca(ctx(), data.data().data(), I(m), I(n),
                       cols_ex ? SVDK_COLUMNS_ARE_EXAMPLES : SVDK_ROWS_ARE_EXAMPLES, method_id(method),
                       I(params.sketch_width), I(params.power_iterations), params.seed.value,
                       center_data ? 1 : 0, basis.data(), eig.data(), &total, mean.data(), &rank));
    PcaModel model;
    const std::size_t r = static_cast<std::size_t>(rank);
    model.basis = take_cols(basis_rows, r, basis);
    model.eigenvalues.assign(eig.begin(), eig.begin() + r);
    model.total_variance = total;
    model.orientation = orientation;
    model.mean = std::move(mean);
    return model;
}

// pca.cpp:118-131
DenseMatrix transform(const PcaModel& model, const DenseMatrix& a) {
    if (model.orientation == Orientation::ColumnsAreExamples) {
        if (a.rows() != model.basis.rows())
            throw DimensionError("transform: data is " + shape_string(a) + " but basis is " +
                                 shape_string(model.basis) + " (feature rows must match)");
        return matmul_transposed_left(model.basis, a);
    }
    if (a.cols() != model.basis.rows())
        throw DimensionError("transform: data is " + shape_string(a) + " but basis is " +
                             shape_string(model.basis) + " (feature columns must match)");
    return matmul(a, model.basis);
}

// pca.cpp:133-168
double residual_delta(const DenseMatrix& a, const SvdResult& s) {
    if (s.u.rows() != a.rows() || s.v.rows() != a.cols())
        throw DimensionError("residual_delta: factors " + shape_string(s.u) + "/" + shape_string(s.v) +
                             " do not match data " + shape_string(a));
    double delta = 0.0;
    check(svdk_residual_delta(ctx(), a.data().data(), I(a.rows()), I(a.cols()), s.u.data().data(),
                              s.sigma.data(), s.v.data().data(), I(s.rank), &delta));
    return delta;
}

}  // namespace svdkit
