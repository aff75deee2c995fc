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

#include <sstream>

#include "svdkit/bench.hpp"
#include "svdkit/cost_model.hpp"
#include "svdkit/csv_io.hpp"
#include "svdkit/dense_matrix.hpp"
#include "svdkit/errors.hpp"
#include "svdkit/idx_io.hpp"
#include "svdkit/kernels.hpp"
#include "svdkit/pca.hpp"
#include "svdkit/svd_methods.hpp"

namespace R = svdkit;  // expands to svdkit_ref under -Dsvdkit=svdkit_ref

namespace {

thread_local double g_residual = 0.0;
thread_local std::size_t g_offset = 0;

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
    } catch (const R::FormatError& e) {
        g_offset = e.offset();
        return 8;
    } catch (const R::IoError&) {
        return 9;
    } catch (...) {
        return 99;
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

// ---- host-side tools: cost model, CSV / IDX formats, bench grid text ----
std::size_t ref_last_offset() { return g_offset; }

int copy_text(const std::string& t, char* out, std::size_t cap) {
    if (t.size() + 1 > cap) return 2;
    std::memcpy(out, t.c_str(), t.size() + 1);
    return 0;
}

// model ids as svdk.h SVDK_COST_*
int ref_cost_model(int model, std::size_t m, std::size_t n, std::size_t l, std::size_t i,
                   double* flops, double* entries, double* bytes) {
    return guard([&] {
        R::CostEstimate c;
        switch (model) {
            case 0: c = R::truncated_cost(m, n); break;
            case 1: c = R::randomized_cost(m, n, l, i); break;
            case 2: c = R::randomized_cost_practical(m, n); break;
            case 3: c = R::krylov_cost(m, n, l, i); break;
            case 4: c = R::krylov_cost_practical(m, n); break;
            case 5: c = R::krylov_cost_per_step(m, n, l, i); break;
            default: throw R::ParamError("model");
        }
        *flops = c.flops;
        *entries = c.space_entries;
        *bytes = c.space_bytes;
    });
}

int ref_format_double(double v, char* out, std::size_t cap) {
    return copy_text(R::format_double(v), out, cap);
}

int ref_idx_parse(const std::uint8_t* bytes, std::size_t len, std::uint64_t* dims) {
    return guard([&] {
        const R::IdxImageSet s = R::parse_idx_images(std::span<const std::uint8_t>(bytes, len));
        dims[0] = s.count;
        dims[1] = s.height;
        dims[2] = s.width;
    });
}

int ref_images_to_matrix(const std::uint8_t* bytes, std::size_t len, double* out) {
    return guard([&] {
        put(R::images_to_matrix(R::parse_idx_images(std::span<const std::uint8_t>(bytes, len))),
            out);
    });
}

int ref_image_as_matrix(const std::uint8_t* bytes, std::size_t len, std::size_t index,
                        double* out) {
    return guard([&] {
        put(R::image_as_matrix(R::parse_idx_images(std::span<const std::uint8_t>(bytes, len)),
                               index),
            out);
    });
}

std::size_t ref_sketch_width_for(double l_fraction, std::size_t n) {
    R::BenchConfig cfg;
    cfg.l_fraction = l_fraction;
    return R::sketch_width_for(cfg, n);
}

// expand_grid: out holds 2 * nr * nc sizes (m, n pairs)
int ref_expand_grid(const std::size_t* rows, std::size_t nr, const std::size_t* cols,
                    std::size_t nc, std::size_t* out, std::size_t* cells) {
    return guard([&] {
        R::BenchConfig cfg;
        cfg.row_sizes.assign(rows, rows + nr);
        cfg.col_sizes.assign(cols, cols + nc);
        cfg.methods = {R::SvdMethod::Truncated};
        const auto g = R::expand_grid(cfg);
        for (std::size_t k = 0; k < g.size(); ++k) {
            out[2 * k] = g[k].first;
            out[2 * k + 1] = g[k].second;
        }
        *cells = g.size();
    });
}

std::vector<R::BenchRecord> records_of(const int* method, const std::size_t* m,
                                       const std::size_t* n, const std::size_t* repeats,
                                       const double* cols5, std::size_t count) {
    // cols5: count x 5 row-major {mean_seconds, std_seconds, delta, model_flops, model_space_bytes}
    std::vector<R::BenchRecord> recs(count);
    for (std::size_t k = 0; k < count; ++k) {
        recs[k].method = static_cast<R::SvdMethod>(method[k]);
        recs[k].m = m[k];
        recs[k].n = n[k];
        recs[k].repeats = repeats[k];
        recs[k].mean_seconds = cols5[5 * k];
        recs[k].std_seconds = cols5[5 * k + 1];
        recs[k].delta = cols5[5 * k + 2];
        recs[k].model_flops = cols5[5 * k + 3];
        recs[k].model_space_bytes = cols5[5 * k + 4];
    }
    return recs;
}

int ref_bench_csv(const int* method, const std::size_t* m, const std::size_t* n,
                  const std::size_t* repeats, const double* cols5, std::size_t count, char* out,
                  std::size_t cap) {
    return copy_text(R::to_csv(records_of(method, m, n, repeats, cols5, count)), out, cap);
}

int ref_ordering_report(const int* method, const std::size_t* m, const std::size_t* n,
                        const std::size_t* repeats, const double* cols5, std::size_t count,
                        char* out, std::size_t cap, double* agreement) {
    const R::OrderingReport r =
        R::summarize_ordering(records_of(method, m, n, repeats, cols5, count));
    *agreement = r.agreement;
    return copy_text(R::format_report(r), out, cap);
}

int ref_matrix_csv_write(const double* a, std::size_t m, std::size_t n, char* out,
                         std::size_t cap) {
    std::ostringstream os;
    R::write_matrix_csv(wrap(a, m, n), os);
    return copy_text(os.str(), out, cap);
}

// read_matrix_csv: out holds up to cap doubles (column-major)
int ref_matrix_csv_read(const char* text, double* out, std::size_t cap, std::size_t* m,
                        std::size_t* n) {
    return guard([&] {
        std::istringstream is{std::string(text)};
        const R::DenseMatrix a = R::read_matrix_csv(is);
        *m = a.rows();
        *n = a.cols();
        if (a.size() > cap) throw R::ParamError("cap");
        put(a, out);
    });
}

}  // extern "C"
