// sketch.cu — randomized PCA and block-Krylov SVD on device.
//
//   randomized_pca  svd_methods.cpp:160-170
//   krylov_svd      svd_methods.cpp:172-196
//   finish_sketch   svd_methods.cpp:97-117 (small_svd + U = Q W + signs)
//
// Same semantics as the reference: Omega is the reference sampler's matrix
// for the seed (host, bit-identical), power iterations H <- A (A^T H) with NO
// re-orthonormalisation in between, Q from qr_thin (CholeskyQR2 here),
// T = A^T Q, then the small SVD of T through the Gram route. Every product
// over the row index is a DMMA GEMM followed (row-sharded) by an allreduce.
#include <algorithm>
#include <thread>
#include <vector>

#include "svdk_methods.h"

namespace svdk {
void gaussian_fill(int64_t rows, int64_t cols, uint64_t seed, double* out);
int64_t qr_thin(Ctx* c, const double* H, int64_t ldh, int64_t m, int64_t p, double* Q, int64_t ldq,
                double* R, const RowComm* comm, double* Rinv_last);

// ---------------------------------------------------------------------------
// Reference Gaussian sampler staged through pinned memory, asynchronously.
// ---------------------------------------------------------------------------
struct HostJob {
    int64_t rows, cols;
    uint64_t seed;
    std::thread th;
};

namespace {
double* staging(Ctx* c, size_t count) {
    if (!c->pinned_ev) SVDK_CUDA(cudaEventCreateWithFlags(&c->pinned_ev, cudaEventDisableTiming));
    // the previous H2D out of the buffer must have landed before we refill it
    SVDK_CUDA(cudaEventSynchronize(c->pinned_ev));
    if (c->pinned_cap < count) {
        if (c->pinned) cudaFreeHost(c->pinned);
        c->pinned = nullptr;
        c->pinned_cap = 0;
        SVDK_CUDA(cudaMallocHost(&c->pinned, sizeof(double) * count));
        c->pinned_cap = count;
    }
    return c->pinned;
}

void join_job(Ctx* c) {
    if (c->omega_job) {
        if (c->omega_job->th.joinable()) c->omega_job->th.join();
        delete c->omega_job;
        c->omega_job = nullptr;
    }
}
}  // namespace

void omega_prefetch(Ctx* c, int64_t rows, int64_t cols, uint64_t seed) {
    join_job(c);
    double* buf = staging(c, static_cast<size_t>(rows) * cols);
    auto* job = new HostJob{rows, cols, seed, {}};
    job->th = std::thread([=] { gaussian_fill(rows, cols, seed, buf); });
    c->omega_job = job;
}

void omega_upload(Ctx* c, int64_t rows, int64_t cols, uint64_t seed, double* d_out, cudaStream_t stream) {
    if (!stream) stream = c->stream;
    const bool ready = c->omega_job && c->omega_job->rows == rows && c->omega_job->cols == cols &&
                       c->omega_job->seed == seed;
    if (ready) {
        join_job(c);
    } else {
        join_job(c);
        gaussian_fill(rows, cols, seed, staging(c, static_cast<size_t>(rows) * cols));
    }
    SVDK_CUDA(cudaMemcpyAsync(d_out, c->pinned, sizeof(double) * rows * cols,
                              cudaMemcpyHostToDevice, stream));
    SVDK_CUDA(cudaEventRecord(c->pinned_ev, stream));
}

void release_host_staging(Ctx* c) {
    join_job(c);
    if (c->pinned_ev) cudaEventSynchronize(c->pinned_ev);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->pinned_ev) cudaEventDestroy(c->pinned_ev);
    c->pinned = nullptr;
    c->pinned_cap = 0;
    c->pinned_ev = nullptr;
}

namespace {

// Y <- A (A^T Y): one power iteration (svd_methods.cpp:165-167).
void power_step(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* Y,
                int64_t ldy, int64_t l, double* Yout, int64_t ldo, double* Z, const RowComm* comm) {
    gemm_tn_rows(c, n, l, m, A, lda, Y, ldy, Z, n, comm);                 // Z = A^T Y
    gemm(c, false, m, l, n, A, lda, Z, n, Yout, ldo, nullptr, true);      // Y = A Z
}

}  // namespace

// svd_methods.cpp:97-117. The orthonormal basis is Q1 Rinv (Q1 m x w
// row-sharded, Rinv w x w upper: CholeskyQR2's implicit last pass), T = A^T Q
// (n x w, replicated).
int64_t finish_sketch(Ctx* c, const double* Q, int64_t ldq, int64_t m, int64_t w, const double* T,
                      int64_t n, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                      const double* Rinv) {
    // The small SVD works on replicated data: no row communicator.
    if (n >= w) {
        const int64_t ldiu = round_up(n, 2);
        DBuf iu(c, static_cast<size_t>(ldiu) * w), iv(c, static_cast<size_t>(w) * w);
        const int64_t r = truncated_svd(c, T, n, n, w, iu.p(), ldiu, sigma, iv.p(), w, nullptr);
        if (r == 0) return 0;
        // normalize_signs first on V = inner.u; U's flips ride on the small
        // factor (Q (-w) = -(Q w) exactly), so U is written once
        copy_mat(c, iu.p(), ldiu, V, ldv, n, r);  // V = inner.u
        DBuf sgn(c, r);
        signs_v(c, V, ldv, n, r, sgn.p());
        DBuf rv(c, static_cast<size_t>(w) * r);  // Rinv inner.v diag(sign) (w x r)
        gemm(c, false, w, r, w, Rinv, w, iv.p(), w, rv.p(), w, sgn.p());
        gemm(c, false, m, r, w, Q, ldq, rv.p(), w, U, ldu, nullptr, true);  // U = Q inner.v
        return r;
    }
    // wide T: factor T^T (w x n) and swap (svd_methods.cpp:100-103)
    const int64_t ldt = round_up(w, 2);
    DBuf Tt(c, static_cast<size_t>(ldt) * n);
    transpose(c, T, n, n, w, Tt.p(), ldt);
    DBuf iu(c, static_cast<size_t>(ldt) * n), iv(c, static_cast<size_t>(n) * n);
    const int64_t r = truncated_svd(c, Tt.p(), ldt, w, n, iu.p(), ldt, sigma, iv.p(), n, nullptr);
    if (r == 0) return 0;
    copy_mat(c, iv.p(), n, V, ldv, n, r);  // V = inner.u
    DBuf sgn(c, r);
    signs_v(c, V, ldv, n, r, sgn.p());
    DBuf rv(c, static_cast<size_t>(w) * r);  // Rinv inner.v diag(sign) (w x r)
    gemm(c, false, w, r, w, Rinv, w, iu.p(), ldt, rv.p(), w, sgn.p());
    gemm(c, false, m, r, w, Q, ldq, rv.p(), w, U, ldu, nullptr, true);  // U = Q inner.v
    return r;
}

int64_t randomized_pca(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t l,
                       int64_t q, uint64_t seed, double* U, int64_t ldu, double* sigma, double* V,
                       int64_t ldv, const RowComm* comm) {
    const int64_t ldh = round_up(std::max<int64_t>(m, 1), 2);
    DBuf H(c, static_cast<size_t>(ldh) * l);
    {
        DBuf Om(c, static_cast<size_t>(n) * l);
        omega_upload(c, n, l, seed, Om.p());
        gemm(c, false, m, l, n, A, lda, Om.p(), n, H.p(), ldh, nullptr, true);  // H = A Omega
    }
    return randomized_from_sketch(c, A, lda, m, n, l, q, std::move(H), ldh, U, ldu, sigma, V, ldv, comm);
}

// The rest of randomized_pca once H = A Omega (m x l, ld ldh) is formed (also
// the entry of the streamed host-buffer path, which forms H chunk by chunk,
// and with Z_first != nullptr the first power iteration's A^T H as well).
int64_t randomized_from_sketch(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t l,
                               int64_t q, DBuf H, int64_t ldh, double* U, int64_t ldu, double* sigma,
                               double* V, int64_t ldv, const RowComm* comm, const double* Z_first) {
    DBuf H2(c, static_cast<size_t>(ldh) * l), Z(c, static_cast<size_t>(n) * l);
    for (int64_t j = 0; j < q; ++j) {
        if (j == 0 && Z_first)  // A^T H already formed by the caller (n x l, ld n)
            gemm(c, false, m, l, n, A, lda, Z_first, n, H2.p(), ldh, nullptr, true);  // H = A Z
        else
            power_step(c, A, lda, m, n, H.p(), ldh, l, H2.p(), ldh, Z.p(), comm);
        std::swap(H, H2);
    }
    // Q = qr_thin(H).q = Q1 Rinv  (H2 reused as Q1)
    DBuf Rinv(c, static_cast<size_t>(l) * l), T(c, static_cast<size_t>(n) * l);
    qr_thin(c, H.p(), ldh, m, l, H2.p(), ldh, nullptr, comm, Rinv.p());
    H.reset();
    gemm_tn_rows(c, n, l, m, A, lda, H2.p(), ldh, Z.p(), n, comm);  // A^T Q1
    gemm(c, false, n, l, l, Z.p(), n, Rinv.p(), l, T.p(), n, nullptr, false, 1.0, false, true);  // T = A^T Q
    return finish_sketch(c, H2.p(), ldh, m, l, T.p(), n, U, ldu, sigma, V, ldv, Rinv.p());
}

int64_t krylov_svd(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t l,
                   int64_t iters, uint64_t seed, double* U, int64_t ldu, double* sigma, double* V,
                   int64_t ldv, const RowComm* comm) {
    const int64_t blocks = iters + 1, w = blocks * l;
    const int64_t ldh = round_up(std::max<int64_t>(m, 1), 2);
    DBuf Om(c, static_cast<size_t>(n) * l), H(c, static_cast<size_t>(ldh) * w),
        Z(c, static_cast<size_t>(n) * std::max(w, l));
    omega_upload(c, n, l, seed, Om.p());
    gemm(c, false, m, l, n, A, lda, Om.p(), n, H.p(), ldh, nullptr, true);  // block 0 = A G
    for (int64_t b = 1; b < blocks; ++b)  // block b = A (A^T block b-1)
        power_step(c, A, lda, m, n, H.p() + (b - 1) * l * ldh, ldh, l, H.p() + b * l * ldh, ldh,
                   Z.p(), comm);
    Om.reset();
    DBuf Q(c, static_cast<size_t>(ldh) * w), Rinv(c, static_cast<size_t>(w) * w),
        T(c, static_cast<size_t>(n) * w);
    qr_thin(c, H.p(), ldh, m, w, Q.p(), ldh, nullptr, comm, Rinv.p());
    H.reset();
    gemm_tn_rows(c, n, w, m, A, lda, Q.p(), ldh, Z.p(), n, comm);  // A^T Q1 (n x w)
    gemm(c, false, n, w, w, Z.p(), n, Rinv.p(), w, T.p(), n, nullptr, false, 1.0, false, true);  // T = A^T Q
    return finish_sketch(c, Q.p(), ldh, m, w, T.p(), n, U, ldu, sigma, V, ldv, Rinv.p());
}

}  // namespace svdk
