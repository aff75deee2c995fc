// synth_host.cpp — host side of the synthetic-input generator (synth.h).
//
// Compiled with -ffp-contract=off -mfma: every floating-point operation is
// the one written (fma() only where spelled out), so these routines give the
// same bits on any x86-64 host and match synth.cu's device kernels. They are
// bench/test input synthesis, not part of the PCA path:
//   svdk_synth_fill       a block of a Gaussian stream (optionally quantised)
//   svdk_synth_add_noise  A += sigma * N   (one rounded product, one rounded sum)
//   svdk_synth_mixing     M = R_X^-1 diag(s) V0^T on a fixed-point grid
// Threads split OUTPUT elements only; each element is produced by one thread
// in a fixed operation order, so the thread count never changes a bit.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#include "svdk.h"
#include "synth.h"

namespace {

int hw_threads() {
    const unsigned h = std::thread::hardware_concurrency();
    return static_cast<int>(std::max(1u, std::min(h, 64u)));
}

// Run body(lo, hi) over [0, count) split into contiguous ranges.
void parallel_for(int64_t count, const std::function<void(int64_t, int64_t)>& body, int64_t grain = 1) {
    const int nt = static_cast<int>(std::min<int64_t>(hw_threads(), std::max<int64_t>(1, count / grain)));
    if (nt <= 1) {
        body(0, count);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(nt);
    for (int t = 0; t < nt; ++t) {
        const int64_t lo = count * t / nt, hi = count * (t + 1) / nt;
        th.emplace_back([&body, lo, hi] { body(lo, hi); });
    }
    for (auto& x : th) x.join();
}

void fill_column(uint64_t seed, uint32_t stream, int quantise, int64_t m_total, int64_t row0, int64_t rows,
                 int64_t j, double* out) {
    const uint64_t e0 = static_cast<uint64_t>(row0) + static_cast<uint64_t>(j) * static_cast<uint64_t>(m_total);
    const uint64_t e1 = e0 + static_cast<uint64_t>(rows);  // exclusive
    for (uint64_t p = e0 >> 1; 2 * p < e1; ++p) {
        double z[2];
        sy_gauss_pair(seed, stream, p, &z[0], &z[1]);
        for (int h = 0; h < 2; ++h) {
            const uint64_t e = 2 * p + h;
            if (e < e0 || e >= e1) continue;
            out[e - e0] = quantise ? sy_quantise_x(z[h]) : z[h];
        }
    }
}

}  // namespace

extern "C" {

int svdk_synth_fill(uint64_t seed, int stream, int quantise, int64_t m_total, int64_t row0, int64_t rows,
                    int64_t cols, double* out, int64_t ld) {
    if (m_total < 0 || row0 < 0 || rows < 0 || cols < 0 || row0 + rows > m_total || ld < rows || !out)
        return SVDK_E_PARAM;
    parallel_for(cols, [&](int64_t lo, int64_t hi) {
        for (int64_t j = lo; j < hi; ++j)
            fill_column(seed, static_cast<uint32_t>(stream), quantise, m_total, row0, rows, j, out + j * ld);
    });
    return SVDK_OK;
}

int svdk_synth_add_noise(uint64_t seed, int64_t m_total, int64_t row0, int64_t rows, int64_t cols, double sigma,
                         double* a, int64_t lda) {
    if (m_total < 0 || row0 < 0 || rows < 0 || cols < 0 || row0 + rows > m_total || lda < rows || !a)
        return SVDK_E_PARAM;
    parallel_for(cols, [&](int64_t lo, int64_t hi) {
        std::vector<double> z(static_cast<size_t>(rows));
        for (int64_t j = lo; j < hi; ++j) {
            fill_column(seed, SY_STREAM_NOISE, 0, m_total, row0, rows, j, z.data());
            double* aj = a + j * lda;
            for (int64_t i = 0; i < rows; ++i) aj[i] = aj[i] + sigma * z[static_cast<size_t>(i)];
        }
    });
    return SVDK_OK;
}

// In-place lower Cholesky of the n x n column-major a (lower triangle used),
// right-looking with column axpys (vectorisable, fixed order per element).
static int chol_lower(double* a, int64_t n) {
    for (int64_t k = 0; k < n; ++k) {
        double* ck = a + k * n;
        if (!(ck[k] > 0.0)) return SVDK_E_NUMERICAL;
        const double d = std::sqrt(ck[k]);
        ck[k] = d;
        for (int64_t i = k + 1; i < n; ++i) ck[i] = ck[i] / d;
        parallel_for(n - k - 1, [&](int64_t lo, int64_t hi) {
            for (int64_t jj = lo; jj < hi; ++jj) {
                const int64_t j = k + 1 + jj;
                const double ljk = ck[j];
                double* cj = a + j * n;
                for (int64_t i = j; i < n; ++i) cj[i] = cj[i] - ljk * ck[i];
            }
        }, 64);
    }
    return SVDK_OK;
}

// Y <- Y L^-T (Y rows x n), i.e. solve Q R = Y with R = L^T; rows are independent.
static void solve_right_lt(const double* l, int64_t n, double* y, int64_t rows, int64_t ldy) {
    parallel_for(rows, [&](int64_t lo, int64_t hi) {
        for (int64_t j = 0; j < n; ++j) {
            double* yj = y + j * ldy;
            for (int64_t k = 0; k < j; ++k) {
                const double rkj = l[j + k * n];  // R(k, j) = L(j, k)
                const double* yk = y + k * ldy;
                for (int64_t i = lo; i < hi; ++i) yj[i] = yj[i] - rkj * yk[i];
            }
            const double d = l[j + j * n];
            for (int64_t i = lo; i < hi; ++i) yj[i] = yj[i] / d;
        }
    }, 16);
}

// G = Y^T Y (n x n, lower triangle filled), Y n_rows x n column-major:
// G(i, j) = sum over rows r ascending of Y(r, i) Y(r, j), via the row-major
// transpose so the inner loop is an axpy over j.
static void gram_lower(const double* y, int64_t rows, int64_t n, double* g) {
    std::vector<double> t(static_cast<size_t>(rows * n));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t r = 0; r < rows; ++r) t[static_cast<size_t>(r * n + j)] = y[r + j * rows];
    std::vector<double> gr(static_cast<size_t>(n * n), 0.0);  // row-major, row i holds G(i, 0..i)
    parallel_for(n, [&](int64_t lo, int64_t hi) {
        for (int64_t r = 0; r < rows; ++r) {
            const double* tr = t.data() + r * n;
            for (int64_t i = lo; i < hi; ++i) {
                const double x = tr[i];
                double* gi = gr.data() + i * n;
                for (int64_t j = 0; j <= i; ++j) gi[j] = gi[j] + x * tr[j];
            }
        }
    }, 8);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j <= i; ++j) g[i + j * n] = gr[static_cast<size_t>(i * n + j)];
}

int svdk_synth_mixing(int64_t n, const double* gx, int64_t ldg, const double* s, uint64_t seed, double* mix,
                      int64_t ldm, double* grid) {
    if (n <= 0 || !gx || !s || !mix || ldg < n || ldm < n) return SVDK_E_PARAM;
    const size_t nn = static_cast<size_t>(n * n);
    // V0 = CholeskyQR2 of the quantised n x n Gaussian (stream V)
    std::vector<double> v(nn), g(nn);
    svdk_synth_fill(seed, SY_STREAM_V, 1, n, 0, n, n, v.data(), n);
    for (int pass = 0; pass < 2; ++pass) {
        gram_lower(v.data(), n, n, g.data());
        if (chol_lower(g.data(), n) != SVDK_OK) return SVDK_E_NUMERICAL;
        solve_right_lt(g.data(), n, v.data(), n, n);
    }
    // R_X = L_X^T from X^T X (exact on every device)
    std::vector<double> lx(nn), r(nn, 0.0);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) lx[static_cast<size_t>(i + j * n)] = gx[i + j * ldg];
    if (chol_lower(lx.data(), n) != SVDK_OK) return SVDK_E_NUMERICAL;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i <= j; ++i) r[static_cast<size_t>(i + j * n)] = lx[static_cast<size_t>(j + i * n)];
    // M = R_X^-1 B, B(i, j) = s_i V0(j, i): column-wise back substitution
    std::vector<double> m(nn);
    parallel_for(n, [&](int64_t lo, int64_t hi) {
        std::vector<double> b(static_cast<size_t>(n));
        for (int64_t j = lo; j < hi; ++j) {
            for (int64_t i = 0; i < n; ++i) b[static_cast<size_t>(i)] = s[i] * v[static_cast<size_t>(j + i * n)];
            double* mj = m.data() + j * n;
            for (int64_t k = n - 1; k >= 0; --k) {
                const double x = b[static_cast<size_t>(k)] / r[static_cast<size_t>(k + k * n)];
                mj[k] = x;
                const double* rk = r.data() + k * n;
                for (int64_t i = 0; i < k; ++i) b[static_cast<size_t>(i)] = b[static_cast<size_t>(i)] - x * rk[i];
            }
        }
    }, 8);
    // fixed-point grid: |M / grid| < 2^B with B = 38 - ceil(log2 n), so any
    // sum of n products x M (|x| < 2^14 units of 2^-10) stays below 2^52 units
    double amax = 0.0;
    for (double x : m) amax = std::max(amax, std::fabs(x));
    if (!(amax > 0.0) || !std::isfinite(amax)) return SVDK_E_NUMERICAL;
    int lg = 0;
    while ((int64_t(1) << lg) < n) ++lg;
    const int B = 38 - lg;
    int E = 0;
    std::frexp(amax, &E);  // amax = f 2^E, f in [0.5, 1)
    const double scale = std::ldexp(1.0, B - E), inv = std::ldexp(1.0, E - B);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i)
            mix[i + j * ldm] = std::nearbyint(m[static_cast<size_t>(i + j * n)] * scale) * inv;
    if (grid) *grid = inv;
    return SVDK_OK;
}

}  // extern "C"
