/*
 * svdk_oracle.c — CPU restatement of the reference svdkit hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see svdk_oracle.h). Each function cites the
 * reference file:line it restates; loop and summation orders are kept so the
 * results are bit-identical to the compiled reference under -ffp-contract=off.
 */
#include "svdk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define AT(p, ld, i, j) (p)[(size_t)(i) + (size_t)(j) * (size_t)(ld)]

/* ---------------------------------------------------------------------- */
/* std::mt19937_64 restated (the C++ standard's parameters).              */
/* ---------------------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i) {
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    const uint64_t MA = 0xB5026F5AA96619E9ULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= MA;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* kernels.cpp:348-379: Box-Muller, cosine first then the sine spare,
 * column-major fill; the spare persists across columns. */
int orc_gaussian_matrix(size_t rows, size_t cols, uint64_t seed, double* out) {
    if (rows < 1 || cols < 1) return ORC_E_PARAM;
    mt64 g;
    mt64_seed(&g, seed);
    int has_spare = 0;
    double spare = 0.0;
    const double pi = 3.141592653589793;
    for (size_t k = 0; k < rows * cols; ++k) {
        if (has_spare) {
            has_spare = 0;
            out[k] = spare;
            continue;
        }
        const double u1 = (double)((mt64_next(&g) >> 11) + 1) * 0x1.0p-53;
        const double u2 = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
        const double radius = sqrt(-2.0 * log(u1));
        const double angle = 2.0 * pi * u2;
        spare = radius * sin(angle);
        has_spare = 1;
        out[k] = radius * cos(angle);
    }
    return ORC_OK;
}

/* kernels.cpp:14-45: jki order, skip b_kj == 0, non-finite -> NumericalError. */
int orc_matmul(const double* a, size_t m, size_t n, const double* b, size_t l, double* c) {
    memset(c, 0, m * l * sizeof(double));
    for (size_t j = 0; j < l; ++j) {
        double* cj = c + j * m;
        const double* bj = b + j * n;
        for (size_t k = 0; k < n; ++k) {
            const double bkj = bj[k];
            if (bkj == 0.0) continue;
            const double* ak = a + k * m;
            for (size_t i = 0; i < m; ++i) cj[i] += ak[i] * bkj;
        }
    }
    for (size_t i = 0; i < m * l; ++i) {
        if (!isfinite(c[i])) return ORC_E_NUMERICAL;
    }
    return ORC_OK;
}

/* kernels.cpp:47-67: c(i,j) = sum_k a(k,i) b(k,j), k ascending. */
int orc_matmul_tl(const double* a, size_t m, size_t n, const double* b, size_t l, double* c) {
    for (size_t j = 0; j < l; ++j) {
        const double* bj = b + j * m;
        for (size_t i = 0; i < n; ++i) {
            const double* ai = a + i * m;
            double sum = 0.0;
            for (size_t k = 0; k < m; ++k) sum += ai[k] * bj[k];
            c[i + j * n] = sum;
        }
    }
    return ORC_OK;
}

/* kernels.cpp:80-97: upper triangle computed, mirrored exactly. */
int orc_gram(const double* a, size_t m, size_t n, double* g) {
    for (size_t j = 0; j < n; ++j) {
        const double* aj = a + j * m;
        for (size_t i = 0; i <= j; ++i) {
            const double* ai = a + i * m;
            double sum = 0.0;
            for (size_t k = 0; k < m; ++k) sum += ai[k] * aj[k];
            AT(g, n, i, j) = sum;
            AT(g, n, j, i) = sum;
        }
    }
    return ORC_OK;
}

/* kernels.cpp:99-105 */
double orc_frobenius_norm_sq(const double* a, size_t count) {
    double sum = 0.0;
    for (size_t i = 0; i < count; ++i) sum += a[i] * a[i];
    return sum;
}

static void transpose(const double* a, size_t m, size_t n, double* t) {
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < m; ++i) AT(t, n, j, i) = AT(a, m, i, j);
}

/* kernels.cpp:111-224: Householder thin QR, drop tol 1e-12 ||h||_F,
 * nonnegative diag(R), explicit Q from reflectors applied in reverse. */
int orc_qr_thin(const double* h, size_t m, size_t p, double* q, double* r, size_t* rank_out) {
    if (m < p) return ORC_E_DIM;
    double* w = (double*)malloc(m * p * sizeof(double));
    memcpy(w, h, m * p * sizeof(double));
    const double drop_tol = 1e-12 * sqrt(orc_frobenius_norm_sq(h, m * p));
    double** vs = (double**)calloc(p ? p : 1, sizeof(double*));
    double* betas = (double*)calloc(p ? p : 1, sizeof(double));
    size_t rank = 0;
    for (size_t k = 0; k < p; ++k) {
        double norm_sq = 0.0;
        for (size_t i = k; i < m; ++i) norm_sq += AT(w, m, i, k) * AT(w, m, i, k);
        const double alpha = sqrt(norm_sq);
        if (alpha <= drop_tol) {
            for (size_t i = k; i < m; ++i) AT(w, m, i, k) = 0.0;
            continue;
        }
        ++rank;
        double* v = (double*)malloc((m - k) * sizeof(double));
        for (size_t i = k; i < m; ++i) v[i - k] = AT(w, m, i, k);
        const double sign = v[0] >= 0.0 ? 1.0 : -1.0;
        v[0] += sign * alpha;
        double vtv = 0.0;
        for (size_t i = 0; i < m - k; ++i) vtv += v[i] * v[i];
        const double beta = 2.0 / vtv;
        vs[k] = v;
        betas[k] = beta;
        for (size_t j = k; j < p; ++j) {
            double dot = 0.0;
            for (size_t i = k; i < m; ++i) dot += v[i - k] * AT(w, m, i, j);
            const double scale = beta * dot;
            for (size_t i = k; i < m; ++i) AT(w, m, i, j) -= scale * v[i - k];
        }
        AT(w, m, k, k) = -sign * alpha;
        for (size_t i = k + 1; i < m; ++i) AT(w, m, i, k) = 0.0;
    }
    double* flip = (double*)malloc((p ? p : 1) * sizeof(double));
    for (size_t k = 0; k < p; ++k) {
        flip[k] = 1.0;
        if (AT(w, m, k, k) < 0.0) {
            flip[k] = -1.0;
            for (size_t j = k; j < p; ++j) AT(w, m, k, j) = -AT(w, m, k, j);
        }
    }
    if (r) {
        memset(r, 0, p * p * sizeof(double));
        for (size_t j = 0; j < p; ++j)
            for (size_t i = 0; i <= j; ++i) AT(r, p, i, j) = AT(w, m, i, j);
    }
    memset(q, 0, m * p * sizeof(double));
    for (size_t j = 0; j < p; ++j) AT(q, m, j, j) = 1.0;
    for (size_t k = p; k-- > 0;) {
        if (betas[k] == 0.0) continue;
        const double* v = vs[k];
        for (size_t j = 0; j < p; ++j) {
            double* qj = q + j * m;
            double dot = 0.0;
            for (size_t i = k; i < m; ++i) dot += v[i - k] * qj[i];
            const double scale = betas[k] * dot;
            for (size_t i = k; i < m; ++i) qj[i] -= scale * v[i - k];
        }
    }
    for (size_t j = 0; j < p; ++j) {
        if (flip[j] < 0.0) {
            double* qj = q + j * m;
            for (size_t i = 0; i < m; ++i) qj[i] = -qj[i];
        }
    }
    for (size_t k = 0; k < p; ++k) free(vs[k]);
    free(vs);
    free(betas);
    free(flip);
    free(w);
    if (rank_out) *rank_out = rank;
    return ORC_OK;
}

/* kernels.cpp:228-237 */
static double off_diagonal_norm(const double* s, size_t n) {
    double sum = 0.0;
    for (size_t j = 0; j < n; ++j)
        for (size_t i = j + 1; i < n; ++i) sum += AT(s, n, i, j) * AT(s, n, i, j);
    return sqrt(2.0 * sum);
}

/* kernels.cpp:241-346: cyclic-by-row Jacobi with the reference's rotation
 * formulas, convergence test and stable descending sort. */
int orc_eig_sym(const double* s, size_t n, int max_sweeps, double* w, double* v,
                double* residual, int* sweeps_done) {
    double max_abs = 0.0, max_asym = 0.0;
    for (size_t j = 0; j < n; ++j) {
        for (size_t i = 0; i < n; ++i) {
            const double x = fabs(AT(s, n, i, j));
            const double y = fabs(AT(s, n, i, j) - AT(s, n, j, i));
            if (max_abs < x) max_abs = x;
            if (max_asym < y) max_asym = y;
        }
    }
    if (max_asym > 1e-8 * max_abs) return ORC_E_PARAM;
    double* a = (double*)malloc((n > 0 ? n * n : 1) * sizeof(double));
    double* vv = (double*)calloc(n > 0 ? n * n : 1, sizeof(double));
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < n; ++i) AT(a, n, i, j) = 0.5 * (AT(s, n, i, j) + AT(s, n, j, i));
    const double threshold = 1e-12 * sqrt(orc_frobenius_norm_sq(a, n * n));
    for (size_t i = 0; i < n; ++i) AT(vv, n, i, i) = 1.0;

    int converged = off_diagonal_norm(a, n) <= threshold;
    int sweep = 0;
    for (; sweep < max_sweeps && !converged; ++sweep) {
        for (size_t p = 0; p + 1 < n; ++p) {
            for (size_t q = p + 1; q < n; ++q) {
                const double apq = AT(a, n, p, q);
                if (apq == 0.0) continue;
                const double tau = (AT(a, n, q, q) - AT(a, n, p, p)) / (2.0 * apq);
                double t;
                if (tau >= 0.0) {
                    t = 1.0 / (tau + sqrt(1.0 + tau * tau));
                } else {
                    t = -1.0 / (-tau + sqrt(1.0 + tau * tau));
                }
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double sn = t * c;
                double* ap = a + p * n;
                double* aq = a + q * n;
                for (size_t i = 0; i < n; ++i) {
                    const double aip = ap[i], aiq = aq[i];
                    ap[i] = c * aip - sn * aiq;
                    aq[i] = sn * aip + c * aiq;
                }
                for (size_t j = 0; j < n; ++j) {
                    const double apj = AT(a, n, p, j), aqj = AT(a, n, q, j);
                    AT(a, n, p, j) = c * apj - sn * aqj;
                    AT(a, n, q, j) = sn * apj + c * aqj;
                }
                AT(a, n, p, q) = 0.0;
                AT(a, n, q, p) = 0.0;
                double* vp = vv + p * n;
                double* vq = vv + q * n;
                for (size_t i = 0; i < n; ++i) {
                    const double vip = vp[i], viq = vq[i];
                    vp[i] = c * vip - sn * viq;
                    vq[i] = sn * vip + c * viq;
                }
            }
        }
        converged = off_diagonal_norm(a, n) <= threshold;
    }
    if (sweeps_done) *sweeps_done = sweep;
    if (!converged) {
        if (residual) *residual = off_diagonal_norm(a, n);
        free(a);
        free(vv);
        return ORC_E_NUMERICAL;
    }
    /* std::stable_sort by descending diagonal: insertion sort is stable. */
    size_t* order = (size_t*)malloc((n ? n : 1) * sizeof(size_t));
    for (size_t i = 0; i < n; ++i) order[i] = i;
    for (size_t i = 1; i < n; ++i) {
        const size_t key = order[i];
        const double kv = AT(a, n, key, key);
        size_t j = i;
        while (j > 0 && kv > AT(a, n, order[j - 1], order[j - 1])) {
            order[j] = order[j - 1];
            --j;
        }
        order[j] = key;
    }
    for (size_t j = 0; j < n; ++j) {
        const size_t src = order[j];
        w[j] = AT(a, n, src, src);
        memcpy(v + j * n, vv + src * n, n * sizeof(double));
    }
    free(order);
    free(a);
    free(vv);
    return ORC_OK;
}

/* svd_methods.cpp:50-71 */
static void normalize_signs(double* u, size_t um, double* v, size_t vn, size_t rank) {
    for (size_t j = 0; j < rank; ++j) {
        double* vj = v + j * vn;
        size_t arg = 0;
        double best = 0.0;
        for (size_t i = 0; i < vn; ++i) {
            if (fabs(vj[i]) > best) {
                best = fabs(vj[i]);
                arg = i;
            }
        }
        if (vj[arg] < 0.0) {
            for (size_t i = 0; i < vn; ++i) vj[i] = -vj[i];
            double* uj = u + j * um;
            for (size_t i = 0; i < um; ++i) uj[i] = -uj[i];
        }
    }
}

/* svd_methods.cpp:121-158 (u m x n, sigma n, v n x n buffers; rank cols valid). */
int orc_truncated_svd(const double* a, size_t m, size_t n, double* u, double* sigma, double* v,
                      size_t* rank_out) {
    if (m < n || n == 0) return ORC_E_DIM;
    double* g = (double*)malloc(n * n * sizeof(double));
    double* w = (double*)malloc(n * sizeof(double));
    double* ev = (double*)malloc(n * n * sizeof(double));
    orc_gram(a, m, n, g);
    double res = 0.0;
    int st = orc_eig_sym(g, n, 30, w, ev, &res, NULL);
    free(g);
    if (st != ORC_OK) {
        free(w);
        free(ev);
        return st;
    }
    for (size_t i = 0; i < n; ++i) sigma[i] = sqrt(w[i] < 0.0 ? 0.0 : w[i]); /* std::max(l, 0.0) */
    size_t rank = 0;
    while (rank < n && sigma[rank] > 1e-12 * sigma[0]) ++rank;
    memcpy(v, ev, n * rank * sizeof(double));
    free(ev);
    free(w);
    st = orc_matmul(a, m, n, v, rank, u);
    if (st != ORC_OK) return st;
    for (size_t j = 0; j < rank; ++j) {
        double* uj = u + j * m;
        const double inv = 1.0 / sigma[j];
        for (size_t i = 0; i < m; ++i) uj[i] *= inv;
    }
    normalize_signs(u, m, v, n, rank);
    *rank_out = rank;
    return ORC_OK;
}

/* svd_methods.cpp:97-117: small SVD of T (n x w) then U = Q W, V = inner U. */
static int finish_sketch(const double* q, size_t m, size_t w, const double* t, size_t n,
                         double* u, double* sigma, double* v, size_t* rank_out) {
    size_t rank = 0;
    double* inner_v; /* the right factor of T (w x rank) */
    int st;
    if (n >= w) {
        double* iu = (double*)malloc(n * w * sizeof(double));
        inner_v = (double*)malloc(w * w * sizeof(double));
        st = orc_truncated_svd(t, n, w, iu, sigma, inner_v, &rank);
        if (st == ORC_OK) memcpy(v, iu, n * rank * sizeof(double));
        free(iu);
    } else {
        double* tt = (double*)malloc(n * w * sizeof(double));
        transpose(t, n, w, tt);
        double* iu = (double*)malloc(w * n * sizeof(double));
        double* iv = (double*)malloc(n * n * sizeof(double));
        st = orc_truncated_svd(tt, w, n, iu, sigma, iv, &rank);
        /* swap_factors: inner.u <- iv (n x r), inner.v <- iu (w x r) */
        if (st == ORC_OK) memcpy(v, iv, n * rank * sizeof(double));
        inner_v = iu;
        free(iv);
        free(tt);
    }
    if (st == ORC_OK) st = orc_matmul(q, m, w, inner_v, rank, u);
    free(inner_v);
    if (st != ORC_OK) return st;
    normalize_signs(u, m, v, n, rank);
    *rank_out = rank;
    return ORC_OK;
}

/* svd_methods.cpp:160-170 */
int orc_randomized_pca(const double* a, size_t m, size_t n, size_t l, size_t q, uint64_t seed,
                       double* u, double* sigma, double* v, size_t* rank) {
    if (m < n || n == 0) return ORC_E_DIM;
    if (l < 1 || l > n) return ORC_E_PARAM;
    double* om = (double*)malloc(n * l * sizeof(double));
    double* h = (double*)malloc(m * l * sizeof(double));
    double* z = (double*)malloc(n * l * sizeof(double));
    orc_gaussian_matrix(n, l, seed, om);
    int st = orc_matmul(a, m, n, om, l, h);
    for (size_t j = 0; j < q && st == ORC_OK; ++j) {
        orc_matmul_tl(a, m, n, h, l, z);
        st = orc_matmul(a, m, n, z, l, h);
    }
    double* qq = (double*)malloc(m * l * sizeof(double));
    if (st == ORC_OK) st = orc_qr_thin(h, m, l, qq, NULL, NULL);
    if (st == ORC_OK) {
        orc_matmul_tl(a, m, n, qq, l, z);
        st = finish_sketch(qq, m, l, z, n, u, sigma, v, rank);
    }
    free(om);
    free(h);
    free(z);
    free(qq);
    return st;
}

/* svd_methods.cpp:172-196 */
int orc_krylov_svd(const double* a, size_t m, size_t n, size_t l, size_t iters, uint64_t seed,
                   double* u, double* sigma, double* v, size_t* rank) {
    if (m < n || n == 0) return ORC_E_DIM;
    if (l < 1 || l > n) return ORC_E_PARAM;
    if (iters < 1) return ORC_E_PARAM;
    const size_t blocks = iters + 1;
    const size_t w = blocks * l;
    if (w > m) return ORC_E_PARAM;
    double* om = (double*)malloc(n * l * sizeof(double));
    double* h = (double*)malloc(m * w * sizeof(double));
    double* z = (double*)malloc(n * (w > l ? w : l) * sizeof(double));
    orc_gaussian_matrix(n, l, seed, om);
    int st = orc_matmul(a, m, n, om, l, h);
    for (size_t b = 1; b < blocks && st == ORC_OK; ++b) {
        orc_matmul_tl(a, m, n, h + (b - 1) * l * m, l, z);
        st = orc_matmul(a, m, n, z, l, h + b * l * m);
    }
    double* qq = (double*)malloc(m * w * sizeof(double));
    if (st == ORC_OK) st = orc_qr_thin(h, m, w, qq, NULL, NULL);
    if (st == ORC_OK) {
        orc_matmul_tl(a, m, n, qq, w, z);
        st = finish_sketch(qq, m, w, z, n, u, sigma, v, rank);
    }
    free(om);
    free(h);
    free(z);
    free(qq);
    return st;
}

/* pca.cpp:13-55 */
int orc_center(const double* a, size_t m, size_t n, int orientation, double* centered,
               double* mean) {
    memcpy(centered, a, m * n * sizeof(double));
    if (orientation == 0) {
        for (size_t i = 0; i < m; ++i) mean[i] = 0.0;
        for (size_t j = 0; j < n; ++j)
            for (size_t i = 0; i < m; ++i) mean[i] += AT(a, m, i, j);
        for (size_t i = 0; i < m; ++i) mean[i] /= (double)n;
        for (size_t j = 0; j < n; ++j)
            for (size_t i = 0; i < m; ++i) AT(centered, m, i, j) -= mean[i];
    } else {
        for (size_t j = 0; j < n; ++j) {
            double sum = 0.0;
            for (size_t i = 0; i < m; ++i) sum += AT(a, m, i, j);
            const double mu = sum / (double)m;
            mean[j] = mu;
            for (size_t i = 0; i < m; ++i) AT(centered, m, i, j) -= mu;
        }
    }
    return ORC_OK;
}

/* pca.cpp:61-89 */
int orc_select_components(const double* w, size_t count, double total, double threshold,
                          size_t* k) {
    if (!(threshold >= 0.0 && threshold <= 1.0)) return ORC_E_PARAM;
    if (!(total > 0.0)) return ORC_E_PARAM;
    double prev = INFINITY;
    for (size_t i = 0; i < count; ++i) {
        if (w[i] < 0.0 || w[i] > prev) return ORC_E_PARAM;
        prev = w[i];
    }
    if (count == 0) return ORC_E_PARAM;
    double cumulative = 0.0;
    for (size_t i = 0; i < count; ++i) {
        cumulative += w[i];
        if (cumulative / total >= threshold) {
            *k = i + 1;
            return ORC_OK;
        }
    }
    *k = 0;
    return ORC_OK;
}
