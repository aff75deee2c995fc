// pca.cu — explained-variance selection and the device PCA pipeline.
//
//   select_components  pca.cpp:61-89
//   fit_pca            pca.cpp:91-116 (RowsAreExamples, device-resident A)
//   center / total     pca.cpp:13-59
#include <algorithm>
#include <cmath>
#include <cstring>

#include "svdk_methods.h"

namespace svdk {
int64_t randomized_pca(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t l,
                       int64_t q, uint64_t seed, double* U, int64_t ldu, double* sigma, double* V,
                       int64_t ldv, const RowComm* comm);
int64_t krylov_svd(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t l,
                   int64_t iters, uint64_t seed, double* U, int64_t ldu, double* sigma, double* V,
                   int64_t ldv, const RowComm* comm);
int64_t lanczos_svd(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t steps,
                    uint64_t seed, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                    const RowComm* comm);

namespace {

// status: 0 ok, 1 bad threshold, 2 bad total, 3 not nonneg-descending, 4 empty.
// out[0] = K (0 = nullopt), out[1] = status, out[2] = total (bits). Validation
// in parallel; the cumulative sum is sequential in index order like the
// reference, so K is decided by the same rounding.
__global__ void select_kernel(const double* w, int64_t count, const double* total_p, double t,
                              int64_t* out) {
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
        const double prev = i == 0 ? INFINITY : w[i - 1];
        if (w[i] < 0.0 || w[i] > prev) bad = 1;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const double total = *total_p;
    int64_t status = 0, k = 0;
    if (!(t >= 0.0 && t <= 1.0))
        status = 1;
    else if (!(total > 0.0))
        status = 2;
    else if (bad)
        status = 3;
    else if (count == 0)
        status = 4;
    else {
        double cumulative = 0.0;
        for (int64_t i = 0; i < count; ++i) {
            cumulative += w[i];
            if (cumulative / total >= t) {
                k = i + 1;
                break;
            }
        }
    }
    out[0] = k;
    out[1] = status;
    out[2] = __double_as_longlong(total);
}

__global__ void square_kernel(const double* s, int64_t r, double* w) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < r;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        w[i] = s[i] * s[i];
}

}  // namespace

// pca.cpp:61-89 with the total variance on the device; returns K (0 =
// nullopt) and optionally the total read back with it (one D2H).
int64_t select_components_dev(Ctx* c, const double* d_w, int64_t count, const double* d_total,
                              double t, double* total_out) {
    DBuf out(c, 3);
    int64_t* o = reinterpret_cast<int64_t*>(out.p());
    select_kernel<<<1, 256, 0, c->stream>>>(d_w, count, d_total, t, o);
    SVDK_CHECK_LAUNCH();
    c->launches++;
    int64_t h[3];
    SVDK_CUDA(cudaMemcpyAsync(h, o, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    SVDK_CUDA(cudaStreamSynchronize(c->stream));
    if (total_out) std::memcpy(total_out, &h[2], sizeof(double));
    switch (h[1]) {
        case 1: {
            char buf[64];
            std::snprintf(buf, sizeof buf, "%f", t);
            fail(SVDK_E_PARAM, std::string("select_components: threshold ") + buf +
                                   " outside [0, 1]");
        }
        case 2:
            fail(SVDK_E_PARAM, "select_components: total variance must be positive");
        case 3:
            fail(SVDK_E_PARAM, "select_components: eigenvalues must be nonnegative descending");
        case 4:
            fail(SVDK_E_PARAM, "select_components: empty spectrum");
        default:
            break;
    }
    return h[0];
}

int64_t select_components(Ctx* c, const double* d_w, int64_t count, double total, double t) {
    DBuf dt(c, 1);
    h2d(c, dt.p(), &total, 1);
    return select_components_dev(c, d_w, count, dt.p(), t, nullptr);
}

namespace {
void dev_pca_body(Ctx* c, const RowComm* comm, const double* A, int64_t m, int64_t n, int64_t lda, int method,
                  int64_t l, int64_t q, uint64_t seed, int center_mode, double threshold, double* U,
                  int64_t ldu, double* sigma, double* V, int64_t ldv, double* mean, int64_t* rank, int64_t* k,
                  double* total);
}  // namespace

void dev_pca(Ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int method, int64_t l,
             int64_t q, uint64_t seed, int center_mode, double threshold, double* U, int64_t ldu,
             double* sigma, double* V, int64_t ldv, double* mean, int64_t* rank, int64_t* k,
             double* total) {
    RowComm rc{c};
    const RowComm* comm = has_comm(c) ? &rc : nullptr;
    // Every rank's arguments are checked locally, then the ranks agree (one
    // small allreduce) so an invalid shard fails on EVERY rank before any
    // data collective instead of leaving its peers waiting.
    int code = 0;
    std::string msg;
    if (m < 0 || n < 0) code = SVDK_E_DIM, msg = "fit_pca: negative dimension";
    else if (lda < std::max<int64_t>(m, 1)) code = SVDK_E_DIM, msg = "fit_pca: lda < rows";
    else if (m > 0 && n > 0 && !A) code = SVDK_E_PARAM, msg = "fit_pca: null A";
    if (comm) {
        // also agree on the replicated arguments (n, method, l, q, centring)
        const double mine[5] = {static_cast<double>(n), static_cast<double>(method), static_cast<double>(l),
                                static_cast<double>(q), static_cast<double>(center_mode)};
        DBuf d(c, 5), s(c, 5);
        h2d(c, d.p(), mine, 5);
        copy_mat(c, d.p(), 5, s.p(), 5, 5, 1);
        comm->broadcast(s.p(), 5, 0);
        double root[5];
        d2h(c, root, s.p(), 5);
        if (!code && std::memcmp(root, mine, sizeof(mine)) != 0)
            code = SVDK_E_PARAM, msg = "fit_pca: n / method / l / q / center differ from rank 0's";
        agree_status(c, comm, code, msg);
    } else if (code) {
        fail(code, msg);
    }
    try {
        dev_pca_body(c, comm, A, m, n, lda, method, l, q, seed, center_mode, threshold, U, ldu, sigma, V, ldv,
                     mean, rank, k, total);
    } catch (const Failure& f) {
        // Validation that depends only on replicated values (n, l, q, global
        // rows) fails identically on every rank; anything else (a CUDA error,
        // a kernel's non-finite flag on one shard) must not strand the peers.
        if (comm && !f.agreed && f.code != SVDK_E_PARAM && f.code != SVDK_E_DIM) abort_comm(c, f.msg);
        throw;
    }
}

namespace {
void dev_pca_body(Ctx* c, const RowComm* comm, const double* A, int64_t m, int64_t n, int64_t lda, int method,
                  int64_t l, int64_t q, uint64_t seed, int center_mode, double threshold, double* U,
                  int64_t ldu, double* sigma, double* V, int64_t ldv, double* mean, int64_t* rank, int64_t* k,
                  double* total) {
    const bool center = center_mode != 0, center_in_place = center_mode == 2;
    const int world = comm ? comm->world() : 1;
    // The reference sampler's Omega (or Lanczos v0) is generated on a host
    // thread while the device centres A and forms the total variance.
    if (method == SVDK_RANDOMIZED || method == SVDK_KRYLOV) {
        if (l >= 1 && l <= n) omega_prefetch(c, n, l, seed);
    } else if (method == SVDK_LANCZOS) {
        omega_prefetch(c, n, 1, seed);
    }
    // global row count
    double mg = static_cast<double>(m);
    if (world > 1) {
        DBuf t(c, 1);
        h2d(c, t.p(), &mg, 1);
        comm->allreduce(t.p(), 1);
        d2h(c, &mg, t.p(), 1);
    }
    if (static_cast<int64_t>(mg) < n || n == 0)
        fail(SVDK_E_DIM, "fit_pca: needs rows >= cols (tall, RowsAreExamples)");
    const int64_t ldc = round_up(std::max<int64_t>(m, 1), 2);
    DBuf C, d_total(c, 1);
    const double* X = A;
    int64_t ldx = lda;
    reset_nonfinite(c);
    if (center) {
        // pca.cpp:37-53: column means over ALL rows, subtract (into a copy, or
        // in place when the caller passed center == 2 and gave up its A)
        if (!center_in_place) C = DBuf(c, static_cast<size_t>(ldc) * n);
        if (world > 1) {
            column_sums(c, A, lda, m, n, 1.0, mean);
            comm->allreduce(mean, static_cast<size_t>(n));
            DBuf sums(c, n);
            copy_mat(c, mean, n, sums.p(), n, n, 1);
            column_sums(c, sums.p(), 1, 1, n, mg, mean);  // mean = sums / m_global
        } else {
            column_sums(c, A, lda, m, n, mg, mean);
        }
        // centring fused with the total variance (pca.cpp:57-59) in one pass
        if (center_in_place) {
            subtract_column_means_sumsq(c, A, lda, m, n, mean, const_cast<double*>(A), lda,
                                        d_total.p());
        } else {
            subtract_column_means_sumsq(c, A, lda, m, n, mean, C.p(), ldc, d_total.p());
            X = C.p();
            ldx = ldc;
        }
        if (comm && world > 1) comm->allreduce(d_total.p(), 1);
    } else {
        fill(c, mean, n, 0.0);
        frob_sq_rows_dev(c, X, ldx, m, n, d_total.p(), comm);  // pca.cpp:57-59
    }
    int64_t r = 0;
    switch (method) {
        case SVDK_TRUNCATED:
            r = truncated_svd(c, X, ldx, m, n, U, ldu, sigma, V, ldv, comm);
            break;
        case SVDK_RANDOMIZED:
            if (l < 1 || l > n) fail(SVDK_E_PARAM, "sketch width l outside [1, n]");
            r = randomized_pca(c, X, ldx, m, n, l, q, seed, U, ldu, sigma, V, ldv, comm);
            break;
        case SVDK_KRYLOV:
            if (l < 1 || l > n) fail(SVDK_E_PARAM, "sketch width l outside [1, n]");
            if (q < 1) fail(SVDK_E_PARAM, "krylov_svd: needs power_iterations >= 1");
            if ((q + 1) * l > static_cast<int64_t>(mg))
                fail(SVDK_E_PARAM, "krylov_svd: block width (i+1)*l exceeds rows");
            r = krylov_svd(c, X, ldx, m, n, l, q, seed, U, ldu, sigma, V, ldv, comm);
            break;
        case SVDK_LANCZOS:
            r = lanczos_svd(c, X, ldx, m, n, l, seed, U, ldu, sigma, V, ldv, comm);
            break;
        default:
            fail(SVDK_E_PARAM, "fit_pca: unknown method");
    }
    *rank = r;
    // eigenvalues = sigma^2 (pca.cpp:111-114), then K (pca.cpp:61-89)
    DBuf w(c, std::max<int64_t>(r, 1));
    if (r > 0) {
        square_kernel<<<static_cast<unsigned>(ceil_div(r, 256)), 256, 0, c->stream>>>(sigma, r,
                                                                                      w.p());
        SVDK_CHECK_LAUNCH();
        c->launches++;
    }
    raise_if_nonfinite(c);
    *k = select_components_dev(c, w.p(), r, d_total.p(), threshold, total);
}
}  // namespace

}  // namespace svdk
