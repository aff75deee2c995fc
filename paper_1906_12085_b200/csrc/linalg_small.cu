// linalg_small.cu — bandwidth-bound helpers around the DMMA engine.
//
//   frob_sq      kernels.cpp:99-105 / pca.cpp:57-59 (total_variance)
//   center_*     pca.cpp:13-55  (column means + subtract, both orientations)
//   transpose    kernels.cpp:69-78
//   copy/fill    layout plumbing (padding to TMA-legal leading dimensions)
//
// All reductions are two-level and fixed-order (per-block partials, then one
// block sums the partials in index order), so results are bit-reproducible
// run to run. These kernels are HBM-bound: one coalesced pass, grid sized to
// a multiple of the SM count.
#include <cmath>

#include "svdk_internal.h"

namespace svdk {
namespace {

__global__ void fill_kernel(double* p, int64_t count, double v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

__global__ void copy_kernel(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                            int64_t cols) {
    for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            dst[i + j * ldd] = src[i + j * lds];
}

__global__ void transpose_kernel(const double* src, int64_t lds, int64_t rows, int64_t cols,
                                 double* dst, int64_t ldd) {
    __shared__ double tile[32][33];
    const int64_t i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t i = i0 + threadIdx.x, j = j0 + k;
        if (i < rows && j < cols) tile[k][threadIdx.x] = src[i + j * lds];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t j = j0 + threadIdx.x, i = i0 + k;  // dst(j, i) = src(i, j)
        if (i < rows && j < cols) dst[j + i * ldd] = tile[threadIdx.x][k];
    }
}

// Per-block partial sums of squares over an m x n block (column-major).
__global__ void sumsq_partial_kernel(const double* A, int64_t lda, int64_t m, int64_t n,
                                     double* partial) {
    __shared__ double red[32];
    double s = 0.0;
    const int64_t total = m * n;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / m, i = e - j * m;
        const double x = A[i + j * lda];
        s = fma(x, x, s);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) partial[blockIdx.x] = s;
    }
}

__global__ void sum_partials_kernel(const double* partial, int count, double* out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) s += partial[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) *out = s;
    }
}

// Column sums over row chunks: grid (n_col_blocks, row_chunks); each block
// handles 32 columns x chunk rows with a warp per column stripe.
constexpr int CS_COLS = 32;
__global__ void colsum_partial_kernel(const double* A, int64_t lda, int64_t m, int64_t n,
                                      int64_t chunk, double* partial /* [chunks][n] */) {
    const int64_t j0 = blockIdx.x * CS_COLS;
    const int64_t r0 = blockIdx.y * chunk, r1 = min(m, r0 + chunk);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int jj = warp; jj < CS_COLS; jj += nw) {
        const int64_t j = j0 + jj;
        if (j >= n) break;
        const double* col = A + j * lda;
        double s = 0.0;
        for (int64_t i = r0 + lane; i < r1; i += 32) s += col[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) partial[blockIdx.y * n + j] = s;
    }
}

__global__ void colsum_finish_kernel(const double* partial, int chunks, int64_t n, double denom,
                                     double* mean) {
    const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int c = 0; c < chunks; ++c) s += partial[c * n + j];
    mean[j] = s / denom;
}

__global__ void sub_colmean_kernel(const double* A, int64_t lda, int64_t m, int64_t n,
                                   const double* mean, double* dst, int64_t ldd) {
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
        const double mu = mean[j];
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            dst[i + j * ldd] = A[i + j * lda] - mu;
    }
}

// dst = A - mean (per column) fused with the sum of squares of the centred
// values (pca.cpp:57-59 total variance) — one HBM pass instead of two.
// Per-block partials, reduced afterwards in fixed order (deterministic).
__global__ void sub_colmean_sumsq_kernel(const double* A, int64_t lda, int64_t m, int64_t n,
                                         const double* mean, double* dst, int64_t ldd,
                                         double* partial) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
        const double mu = mean[j];
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const double x = A[i + j * lda] - mu;
            dst[i + j * ldd] = x;
            s = fma(x, x, s);
        }
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (blockDim.x >> 5); ++w) s += red[w];
        partial[blockIdx.x + static_cast<int64_t>(blockIdx.y) * gridDim.x] = s;
    }
}

// Row means (ColumnsAreExamples): mean_i = sum_j a_ij / n, j ascending.
__global__ void rowmean_kernel(const double* A, int64_t lda, int64_t m, int64_t n, double* mean) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= m) return;
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) s += A[i + j * lda];
    mean[i] = s / static_cast<double>(n);
}

__global__ void sub_rowmean_kernel(const double* A, int64_t lda, int64_t m, int64_t n,
                                   const double* mean, double* dst, int64_t ldd) {
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            dst[i + j * ldd] = A[i + j * lda] - mean[i];
}

__global__ void scale_rows_kernel(double* W, int64_t ldw, int64_t rows, int64_t cols,
                                  const double* s) {
    for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            W[i + j * ldw] *= s[i];
}

dim3 grid2d(Ctx* c, int64_t rows, int64_t cols, int threads) {
    int64_t gx = std::min<int64_t>(ceil_div(rows, threads), 4 * c->num_sms);
    int64_t gy = std::min<int64_t>(cols, 65535);
    if (gx < 1) gx = 1;
    if (gy < 1) gy = 1;
    return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
}

}  // namespace

void scale_rows(Ctx* c, double* W, int64_t ldw, int64_t rows, int64_t cols, const double* s) {
    if (rows <= 0 || cols <= 0) return;
    scale_rows_kernel<<<grid2d(c, rows, cols, 256), 256, 0, c->stream>>>(W, ldw, rows, cols, s);
    SVDK_CHECK_LAUNCH();
    c->launches++;
}

__global__ void identity_kernel(double* X, int64_t ld, int64_t n) {
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            X[i + j * ld] = i == j ? 1.0 : 0.0;
}

void set_identity(Ctx* c, double* X, int64_t ld, int64_t n) {
    if (n <= 0) return;
    identity_kernel<<<grid2d(c, n, n, 256), 256, 0, c->stream>>>(X, ld, n);
    SVDK_CHECK_LAUNCH();
    c->launches++;
}

void fill(Ctx* c, double* p, int64_t count, double v) {
    if (count <= 0) return;
    const int64_t blocks = std::min<int64_t>(ceil_div(count, 256), 8 * c->num_sms);
    fill_kernel<<<static_cast<unsigned>(blocks), 256, 0, c->stream>>>(p, count, v);
    SVDK_CHECK_LAUNCH();
    c->launches++;
}

void copy_mat(Ctx* c, const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
              int64_t cols) {
    if (rows <= 0 || cols <= 0) return;
    if (lds == rows && ldd == rows) {
        SVDK_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * rows * cols, cudaMemcpyDeviceToDevice,
                                  c->stream));
        return;
    }
    copy_kernel<<<grid2d(c, rows, cols, 256), 256, 0, c->stream>>>(src, lds, dst, ldd, rows, cols);
    SVDK_CHECK_LAUNCH();
    c->launches++;
}

void transpose(Ctx* c, const double* src, int64_t lds, int64_t rows, int64_t cols, double* dst,
               int64_t ldd) {
    if (rows <= 0 || cols <= 0) return;
    dim3 grid(static_cast<unsigned>(ceil_div(rows, 32)), static_cast<unsigned>(ceil_div(cols, 32)));
    transpose_kernel<<<grid, dim3(32, 8), 0, c->stream>>>(src, lds, rows, cols, dst, ldd);
    SVDK_CHECK_LAUNCH();
    c->launches++;
}

void frob_sq_dev(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, double* d_out) {
    if (m <= 0 || n <= 0) {
        fill(c, d_out, 1, 0.0);
        return;
    }
    const int blocks = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(ceil_div(m * n, 256), 4 * c->num_sms)));
    DBuf partial(c, blocks);
    sumsq_partial_kernel<<<blocks, 256, 0, c->stream>>>(A, lda, m, n, partial.p());
    SVDK_CHECK_LAUNCH();
    sum_partials_kernel<<<1, 256, 0, c->stream>>>(partial.p(), blocks, d_out);
    SVDK_CHECK_LAUNCH();
    c->launches += 2;
}

double frob_sq(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n) {
    DBuf t(c, 1);
    frob_sq_dev(c, A, lda, m, n, t.p());
    double out = 0.0;
    d2h(c, &out, t.p(), 1);
    return out;
}

void column_sums(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, double denom,
                 double* d_out) {
    const int64_t colblocks = ceil_div(n, CS_COLS);
    int64_t chunks = std::max<int64_t>(1, (4 * c->num_sms + colblocks - 1) / colblocks);
    int64_t chunk = round_up(ceil_div(std::max<int64_t>(m, 1), chunks), 32);
    chunks = std::max<int64_t>(1, ceil_div(std::max<int64_t>(m, 1), chunk));
    DBuf partial(c, static_cast<size_t>(chunks) * n);
    colsum_partial_kernel<<<dim3(static_cast<unsigned>(colblocks), static_cast<unsigned>(chunks)),
                            256, 0, c->stream>>>(A, lda, m, n, chunk, partial.p());
    SVDK_CHECK_LAUNCH();
    colsum_finish_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c->stream>>>(
        partial.p(), static_cast<int>(chunks), n, denom, d_out);
    SVDK_CHECK_LAUNCH();
    c->launches += 2;
}

void subtract_column_means(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n,
                           const double* d_mean, double* dst, int64_t ldd) {
    if (m <= 0 || n <= 0) return;
    sub_colmean_kernel<<<grid2d(c, m, n, 256), 256, 0, c->stream>>>(A, lda, m, n, d_mean, dst,
                                                                     ldd);
    SVDK_CHECK_LAUNCH();
    c->launches++;
}

void subtract_column_means_sumsq(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n,
                                 const double* d_mean, double* dst, int64_t ldd, double* d_sumsq) {
    if (m <= 0 || n <= 0) {
        fill(c, d_sumsq, 1, 0.0);
        return;
    }
    // fewer column blocks than the plain subtract so the partials stay small
    const dim3 g(static_cast<unsigned>(std::min<int64_t>(ceil_div(m, 256), 2 * c->num_sms)),
                 static_cast<unsigned>(std::min<int64_t>(n, 256)));
    DBuf partial(c, static_cast<size_t>(g.x) * g.y);
    sub_colmean_sumsq_kernel<<<g, 256, 0, c->stream>>>(A, lda, m, n, d_mean, dst, ldd, partial.p());
    SVDK_CHECK_LAUNCH();
    sum_partials_kernel<<<1, 256, 0, c->stream>>>(partial.p(), static_cast<int>(g.x * g.y), d_sumsq);
    SVDK_CHECK_LAUNCH();
    c->launches += 2;
}

void center_rows_are_examples(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n,
                              double* dst, int64_t ldd, double* d_mean) {
    const int64_t colblocks = ceil_div(n, CS_COLS);
    // enough row chunks to fill the machine, chunk a multiple of 32
    int64_t chunks = std::max<int64_t>(1, (4 * c->num_sms + colblocks - 1) / colblocks);
    int64_t chunk = round_up(ceil_div(m, chunks), 32);
    chunks = std::max<int64_t>(1, ceil_div(m, chunk));
    DBuf partial(c, static_cast<size_t>(chunks) * n);
    colsum_partial_kernel<<<dim3(static_cast<unsigned>(colblocks), static_cast<unsigned>(chunks)),
                            256, 0, c->stream>>>(A, lda, m, n, chunk, partial.p());
    SVDK_CHECK_LAUNCH();
    colsum_finish_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c->stream>>>(
        partial.p(), static_cast<int>(chunks), n, static_cast<double>(m), d_mean);
    SVDK_CHECK_LAUNCH();
    sub_colmean_kernel<<<grid2d(c, m, n, 256), 256, 0, c->stream>>>(A, lda, m, n, d_mean, dst,
                                                                     ldd);
    SVDK_CHECK_LAUNCH();
    c->launches += 3;
}

void center_cols_are_examples(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n,
                              double* dst, int64_t ldd, double* d_mean) {
    rowmean_kernel<<<static_cast<unsigned>(ceil_div(m, 256)), 256, 0, c->stream>>>(A, lda, m, n,
                                                                                   d_mean);
    SVDK_CHECK_LAUNCH();
    sub_rowmean_kernel<<<grid2d(c, m, n, 256), 256, 0, c->stream>>>(A, lda, m, n, d_mean, dst,
                                                                     ldd);
    SVDK_CHECK_LAUNCH();
    c->launches += 2;
}

}  // namespace svdk
