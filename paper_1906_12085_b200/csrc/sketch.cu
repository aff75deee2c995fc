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
#include <vector>

#include "svdk_methods.h"

namespace svdk {
void gaussian_fill(int64_t rows, int64_t cols, uint64_t seed, double* out);
int64_t qr_thin(Ctx* c, const double* H, int64_t ldh, int64_t m, int64_t p, double* Q, int64_t ldq,
                double* R, const RowComm* comm);

namespace {

// Omega (n x l) from the reference sampler, uploaded through pinned memory.
void upload_omega(Ctx* c, int64_t n, int64_t l, uint64_t seed, double* dO) {
    double* h = nullptr;
    SVDK_CUDA(cudaMallocHost(&h, sizeof(double) * n * l));
    gaussian_fill(n, l, seed, h);
    SVDK_CUDA(cudaMemcpyAsync(dO, h, sizeof(double) * n * l, cudaMemcpyHostToDevice, c->stream));
    SVDK_CUDA(cudaStreamSynchronize(c->stream));
    cudaFreeHost(h);
}

// Y <- A (A^T Y): one power iteration (svd_methods.cpp:165-167).
void power_step(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* Y,
                int64_t ldy, int64_t l, double* Yout, int64_t ldo, double* Z, const RowComm* comm) {
    gemm_tn_rows(c, n, l, m, A, lda, Y, ldy, Z, n, comm);                 // Z = A^T Y
    gemm(c, false, m, l, n, A, lda, Z, n, Yout, ldo, nullptr, true);      // Y = A Z
}

}  // namespace

// svd_methods.cpp:97-117. Q (m x w, row-sharded), T = A^T Q (n x w, replicated).
int64_t finish_sketch(Ctx* c, const double* Q, int64_t ldq, int64_t m, int64_t w, const double* T,
                      int64_t n, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv) {
    // The small SVD works on replicated data: no row communicator.
    if (n >= w) {
        const int64_t ldiu = round_up(n, 2);
        DBuf iu(c, static_cast<size_t>(ldiu) * w), iv(c, static_cast<size_t>(w) * w);
        const int64_t r = truncated_svd(c, T, n, n, w, iu.p(), ldiu, sigma, iv.p(), w, nullptr);
        if (r == 0) return 0;
        reset_nonfinite(c);
        gemm(c, false, m, r, w, Q, ldq, iv.p(), w, U, ldu, nullptr, true);  // U = Q inner.v
        raise_if_nonfinite(c);
        copy_mat(c, iu.p(), ldiu, V, ldv, n, r);                             // V = inner.u
        normalize_signs_uv(c, U, ldu, m, V, ldv, n, r);
        return r;
    }
    // wide T: factor T^T (w x n) and swap (svd_methods.cpp:100-103)
    const int64_t ldt = round_up(w, 2);
    DBuf Tt(c, static_cast<size_t>(ldt) * n);
    transpose(c, T, n, n, w, Tt.p(), ldt);
    DBuf iu(c, static_cast<size_t>(ldt) * n), iv(c, static_cast<size_t>(n) * n);
    const int64_t r = truncated_svd(c, Tt.p(), ldt, w, n, iu.p(), ldt, sigma, iv.p(), n, nullptr);
    if (r == 0) return 0;
    reset_nonfinite(c);
    gemm(c, false, m, r, w, Q, ldq, iu.p(), ldt, U, ldu, nullptr, true);  // U = Q inner.v
    raise_if_nonfinite(c);
    copy_mat(c, iv.p(), n, V, ldv, n, r);                                  // V = inner.u
    normalize_signs_uv(c, U, ldu, m, V, ldv, n, r);
    return r;
}

int64_t randomized_pca(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t l,
                       int64_t q, uint64_t seed, double* U, int64_t ldu, double* sigma, double* V,
                       int64_t ldv, const RowComm* comm) {
    const int64_t ldh = round_up(std::max<int64_t>(m, 1), 2);
    DBuf Om(c, static_cast<size_t>(n) * l), H(c, static_cast<size_t>(ldh) * l),
        H2(c, static_cast<size_t>(ldh) * l), Z(c, static_cast<size_t>(n) * l);
    upload_omega(c, n, l, seed, Om.p());
    reset_nonfinite(c);
    gemm(c, false, m, l, n, A, lda, Om.p(), n, H.p(), ldh, nullptr, true);  // H = A Omega
    for (int64_t j = 0; j < q; ++j) {
        power_step(c, A, lda, m, n, H.p(), ldh, l, H2.p(), ldh, Z.p(), comm);
        std::swap(H, H2);
    }
    raise_if_nonfinite(c);
    Om.reset();
    // Q = qr_thin(H).q  (H2 reused as Q)
    qr_thin(c, H.p(), ldh, m, l, H2.p(), ldh, nullptr, comm);
    H.reset();
    gemm_tn_rows(c, n, l, m, A, lda, H2.p(), ldh, Z.p(), n, comm);  // T = A^T Q
    return finish_sketch(c, H2.p(), ldh, m, l, Z.p(), n, U, ldu, sigma, V, ldv);
}

int64_t krylov_svd(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t l,
                   int64_t iters, uint64_t seed, double* U, int64_t ldu, double* sigma, double* V,
                   int64_t ldv, const RowComm* comm) {
    const int64_t blocks = iters + 1, w = blocks * l;
    const int64_t ldh = round_up(std::max<int64_t>(m, 1), 2);
    DBuf Om(c, static_cast<size_t>(n) * l), H(c, static_cast<size_t>(ldh) * w),
        Z(c, static_cast<size_t>(n) * std::max(w, l));
    upload_omega(c, n, l, seed, Om.p());
    reset_nonfinite(c);
    gemm(c, false, m, l, n, A, lda, Om.p(), n, H.p(), ldh, nullptr, true);  // block 0 = A G
    for (int64_t b = 1; b < blocks; ++b)  // block b = A (A^T block b-1)
        power_step(c, A, lda, m, n, H.p() + (b - 1) * l * ldh, ldh, l, H.p() + b * l * ldh, ldh,
                   Z.p(), comm);
    raise_if_nonfinite(c);
    Om.reset();
    DBuf Q(c, static_cast<size_t>(ldh) * w);
    qr_thin(c, H.p(), ldh, m, w, Q.p(), ldh, nullptr, comm);
    H.reset();
    gemm_tn_rows(c, n, w, m, A, lda, Q.p(), ldh, Z.p(), n, comm);  // T = A^T Q (n x w)
    return finish_sketch(c, Q.p(), ldh, m, w, Z.p(), n, U, ldu, sigma, V, ldv);
}

}  // namespace svdk
