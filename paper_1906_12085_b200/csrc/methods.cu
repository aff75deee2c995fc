// methods.cu — device orchestration of the SVD methods and PCA steps.
//
//   truncated_svd   svd_methods.cpp:121-158
//   normalize_signs svd_methods.cpp:50-71   (folded into the U epilogue scale)
//   select          pca.cpp:61-89
//
// Everything runs on the context stream with device-resident operands; the
// host only reads back scalars it needs for control flow (rank, K, status).
#include <algorithm>
#include <cmath>

#include "svdk_methods.h"

namespace svdk {
namespace {

// sigma_i = sqrt(max(l_i, 0)) ; rank = first i with !(sigma_i > 1e-12 sigma_0).
__global__ void spectrum_kernel(const double* w, int64_t n, double* sigma, int* rank_out) {
    __shared__ int first_bad;
    if (threadIdx.x == 0) first_bad = static_cast<int>(n);
    __syncthreads();
    const double l0 = w[0];
    const double s0 = sqrt(l0 < 0.0 ? 0.0 : l0);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double l = w[i];
        const double s = sqrt(l < 0.0 ? 0.0 : l);  // std::max(l, 0.0) keeps -0.0
        sigma[i] = s;
        if (!(s > 1e-12 * s0)) atomicMin(&first_bad, static_cast<int>(i));
    }
    __syncthreads();
    if (threadIdx.x == 0) *rank_out = first_bad;
}

// One warp per column j < rank: first index of max |v_ij| (strict >), then
// sign flip of V_j and epilogue scale_j = sign_j * (1 / sigma_j) for U.
__global__ void signs_kernel(double* V, int64_t ldv, int64_t n, const int* rank_p, int rank_val,
                             const double* sigma, double* scale, int with_scale) {
    const int rank = rank_p ? *rank_p : rank_val;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= rank) return;
    double* v = V + warp * ldv;
    double best = 0.0;
    int64_t arg = 0;
    for (int64_t i = lane; i < n; i += 32) {
        const double a = fabs(v[i]);
        if (a > best) {
            best = a;
            arg = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int64_t oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (ob > best || (ob == best && oa < arg)) {
            best = ob;
            arg = oa;
        }
    }
    // lanes that never saw a positive |v| keep arg = 0 with best = 0: consistent
    // with the reference (arg stays 0 when the column is all zero).
    const double pivot = v[arg];
    const double sign = pivot < 0.0 ? -1.0 : 1.0;
    if (sign < 0.0)
        for (int64_t i = lane; i < n; i += 32) v[i] = -v[i];
    // U is formed from the already-flipped V: A(-v) = -(Av) exactly, so
    // scaling by 1/sigma reproduces the reference's flip-after-scale.
    if (with_scale == 1 && lane == 0) scale[warp] = 1.0 / sigma[warp];
    if (with_scale == 2 && lane == 0) scale[warp] = sign;  // the sketch methods' U flip
}

}  // namespace

void raise_if_nonfinite(Ctx* c) {
    int flag = 0;
    SVDK_CUDA(cudaMemcpyAsync(&flag, c->d_flags, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    SVDK_CUDA(cudaStreamSynchronize(c->stream));
    if (flag) {
        SVDK_CUDA(cudaMemsetAsync(c->d_flags, 0, sizeof(int), c->stream));
        fail(SVDK_E_NUMERICAL, "matmul: non-finite result (overflow)", 0.0);
    }
}

void reset_nonfinite(Ctx* c) {
    SVDK_CUDA(cudaMemsetAsync(c->d_flags, 0, sizeof(int), c->stream));
}

int64_t spectrum(Ctx* c, const double* w, int64_t n, double* sigma) {
    spectrum_kernel<<<1, 1024, 0, c->stream>>>(w, n, sigma, c->d_flags + 2);
    SVDK_CHECK_LAUNCH();
    c->launches++;
    int rank = 0;
    SVDK_CUDA(cudaMemcpyAsync(&rank, c->d_flags + 2, sizeof(int), cudaMemcpyDeviceToHost,
                              c->stream));
    SVDK_CUDA(cudaStreamSynchronize(c->stream));
    return rank;
}

void signs_v(Ctx* c, double* V, int64_t ldv, int64_t n, int64_t rank, double* d_sign) {
    if (rank <= 0) return;
    signs_kernel<<<static_cast<unsigned>(ceil_div(rank * 32, 256)), 256, 0, c->stream>>>(
        V, ldv, n, nullptr, static_cast<int>(rank), nullptr, d_sign, 2);
    SVDK_CHECK_LAUNCH();
    c->launches++;
}

// svd_methods.cpp:127-156: from eigenpairs (w descending, Vfull n x kcols)
// of A^T A to sigma, the numerical rank, sign-normalised V and U = A V / sigma.
int64_t back_project(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* w,
                     const double* Vfull, int64_t ldvf, int64_t kcols, double* U, int64_t ldu,
                     double* sigma, double* V, int64_t ldv) {
    const int64_t rank = spectrum(c, w, kcols, sigma);
    if (rank == 0) return 0;
    copy_mat(c, Vfull, ldvf, V, ldv, n, rank);
    DBuf scale(c, rank);
    const int warps = static_cast<int>(rank);
    signs_kernel<<<static_cast<unsigned>(ceil_div(warps * 32, 256)), 256, 0, c->stream>>>(
        V, ldv, n, c->d_flags + 2, 0, sigma, scale.p(), 1);
    SVDK_CHECK_LAUNCH();
    c->launches++;
    // U = A V diag(1 / sigma) on the sign-normalised V (kernels.cpp:14-45 +
    // svd_methods.cpp:146-156); non-finite products set the sticky flag.
    gemm(c, false, m, rank, n, A, lda, V, ldv, U, ldu, scale.p(), true);
    return rank;
}

// svd_methods.cpp:121-158 on device. A m x n (m >= n checked by caller).
// Outputs: U (m x rank, ldu), sigma (n entries written, rank valid),
// V (n x rank, ldv). Returns rank.
int64_t truncated_svd(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, double* U,
                      int64_t ldu, double* sigma, double* V, int64_t ldv, const RowComm* comm) {
    DBuf G(c, static_cast<size_t>(n) * n);
    gram_rows(c, A, lda, m, n, G.p(), n, comm);
    return truncated_from_gram(c, A, lda, m, n, std::move(G), U, ldu, sigma, V, ldv, comm);
}

// The rest of truncated_svd once G = A^T A (n x n, ld n) is formed (also the
// entry of the streamed host-buffer path, which accumulates G chunk by chunk).
int64_t truncated_from_gram(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, DBuf G,
                            double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                            const RowComm* comm) {
    DBuf w(c, n), Vfull(c, static_cast<size_t>(n) * n);
    eig_sym_rows(c, G.p(), n, n, w.p(), Vfull.p(), n, comm);
    G.reset();
    return back_project(c, A, lda, m, n, w.p(), Vfull.p(), n, n, U, ldu, sigma, V, ldv);
}

}  // namespace svdk
