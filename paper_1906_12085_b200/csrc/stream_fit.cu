// stream_fit.cu — fit_pca from a HOST buffer with the upload streamed under
// the first pass over A (reference pca.cpp:91-116 + svd_methods.cpp:121-170).
//
// svdk_fit_pca's plain path copies all of A to the GPU, then centres it, then
// runs the method: the PCIe copy (30 ms at c2, 1.2 s at c4) and the first pass
// over A (the Gram for truncated, H = A Omega for randomized) run back to back.
// Here A arrives in chunks on a copy stream, and the compute stream works on
// the chunks that have landed. Truncated uses COLUMN chunks: a chunk holds
// whole columns, so it is centred exactly as the reference centres the matrix
// (column mean, then subtract, pca.cpp:37-53, fused with the chunk's sum of
// squares for the total variance), and then contributes its block column of
// the Gram:
//   G[0:j1, j0:j1] = A[:, 0:j1]^T A[:, j0:j1]
// (the upper triangle is mirrored at the end, as the reference's gram
// computes i <= j and mirrors, kernels.cpp:80-97).
// Randomized uses ROW chunks instead (H = A Omega is row-separable; see
// streamed_sketch_rows). The rest of the method then runs on the resident,
// centred A.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "svdk_methods.h"

namespace svdk {
namespace {

// G[j, i] = G[i, j] for i < j (upper triangle authoritative).
__global__ void mirror_upper_kernel(double* G, int64_t ldg, int64_t n) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / n, i = e - j * n;
        if (i > j) G[i + j * ldg] = G[j + i * ldg];
    }
}

// Row-chunk path (randomized): mu = sum_k cnt_k mu_k / m (chunk order) and
// d_k = mu_k - mu (C x n, ld ldd), from the per-chunk column means mu_k.
__global__ void chunk_means_kernel(const double* mu_k /* [C][n] */, int C, int64_t n, int64_t rows,
                                   int64_t m, double* mu, double* d, int64_t ldd) {
    const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int k = 0; k < C; ++k) s = fma(static_cast<double>(min(rows, m - k * rows)), mu_k[k * n + j], s);
    const double mj = s / static_cast<double>(m);
    mu[j] = mj;
    for (int k = 0; k < C; ++k) d[k + j * ldd] = mu_k[k * n + j] - mj;
}

// X[i, j] += Y[i / rows, j] (the offset row of i's chunk), m x w; with
// partial != nullptr also the per-CTA sums of squares of the result.
__global__ void add_chunk_rows_kernel(double* X, int64_t ldx, int64_t m, int64_t w, const double* Y,
                                      int64_t ldy, int64_t rows, double* partial) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t j = blockIdx.y; j < w; j += gridDim.y) {
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const double x = X[i + j * ldx] + Y[i / rows + j * ldy];
            X[i + j * ldx] = x;
            s = fma(x, x, s);
        }
    }
    if (!partial) return;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (blockDim.x >> 5); ++k) s += red[k];
        partial[blockIdx.x + static_cast<int64_t>(blockIdx.y) * gridDim.x] = s;
    }
}

// E[k, j] = SH[k][j] + cnt_k W[k, j] (C x l, ld ldd; padding rows zero): the
// chunk-sum term of the first power iteration's correction (see below).
__global__ void sketch_corr_kernel(const double* SH /* [C][l] */, const double* W, int C, int64_t l,
                                   int64_t rows, int64_t m, int64_t ldd, double* E) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < ldd * l;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / ldd, k = e - j * ldd;
        double v = 0.0;
        if (k < C) v = fma(static_cast<double>(min(rows, m - k * rows)), W[k + j * ldd], SH[k * l + j]);
        E[k + j * ldd] = v;
    }
}

__global__ void sum_fixed_order_kernel(const double* partial, int count, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < count; ++i) s += partial[i];
        *out = s;
    }
}

// Columns per chunk for the Gram (~n/8, a multiple of 64 so chunks stay
// TMA-aligned; each block column of G is written once); 0 = do not stream
// (fewer than 2 chunks, or too little data to matter).
int64_t chunk_cols(int64_t m, int64_t n) {
    if (const char* e = std::getenv("SVDK_STREAM_COLS")) {  // test / tuning override
        const int64_t v = std::atoll(e);
        return v <= 0 ? 0 : round_up(std::max<int64_t>(v, 64), 64);
    }
    if (8.0 * static_cast<double>(m) * static_cast<double>(n) < 64.0 * (1 << 20)) return 0;
    return round_up(std::max<int64_t>(ceil_div(n, 8), 64), 64);
}

// Rows per chunk for the sketch (~256 MB of A, a multiple of 64 rows); 0 = do not stream.
int64_t chunk_rows(int64_t m, int64_t n) {
    if (const char* e = std::getenv("SVDK_STREAM_ROWS")) {  // test / tuning override
        const int64_t v = std::atoll(e);
        return v <= 0 ? 0 : round_up(std::max<int64_t>(v, 64), 64);
    }
    const int64_t r = round_up(std::max<int64_t>((int64_t{256} << 20) / (8 * std::max<int64_t>(n, 1)), 1024), 64);
    return m >= 2 * r ? r : 0;
}

// Randomized, row chunks (a row chunk of the column-major host buffer is one
// 2-D DMA, n runs of rows*8 bytes: measured at the contiguous rate, 55.6 GB/s,
// tools/probes/h2d2d.cu). H = A^c Omega is row-separable, but the global
// column means are only known at the end, so each chunk is centred by ITS OWN
// means mu_k and the difference is added back in closed form (the pairwise
// update of Chan, Golub & LeVeque applied to the product):
//   A^c rows of chunk k = (A_k - 1 mu_k^T) + 1 d_k^T,  d_k = mu_k - mu,
//   H rows of chunk k   = (A_k - 1 mu_k^T) Omega + 1 (Omega^T d_k)^T.
// d_k is the spread of the chunk means, so the correction introduces no
// cancellation. With power iterations (q >= 1) the first A^T H is accumulated
// per chunk as well, Z = sum_k (A_k - 1 mu_k^T)^T H_k^raw, and corrected with
//   A^c^T H = Z + sum_k d_k (s_k + cnt_k w_k)^T,  s_k = H_k^raw^T 1, w_k = Omega^T d_k
// (the (A_k - 1 mu_k^T)^T 1 terms vanish: each chunk is centred by its own
// mean). One more pass adds d_k to the stored chunks (A becomes the globally
// centred matrix the remaining iterations read), fused with the total.
bool streamed_sketch_rows(Ctx* c, const double* host, int64_t m, int64_t n, int64_t l, int64_t q, uint64_t seed,
                          double* basis, double* eigenvalues, double* total, double* mean, int64_t* rank) {
    const int64_t rows = chunk_rows(m, n);
    if (rows <= 0 || rows >= m) return false;
    validate_method(SVDK_RANDOMIZED, m, n, l, q, "fit_pca");
    const int64_t C = ceil_div(m, rows);
    cudaStream_t S = c->stream;
    int64_t lda;
    DBuf dA = alloc_mat(c, m, n, lda);
    DBuf mu_k(c, static_cast<size_t>(C) * n), mu(c, n);
    const int64_t ldh = round_up(m, 2);
    DBuf H(c, static_cast<size_t>(ldh) * l), Om(c, static_cast<size_t>(n) * l);
    const bool with_z = q >= 1;
    DBuf Z(c, with_z ? static_cast<size_t>(n) * l : 1), SH(c, with_z ? static_cast<size_t>(C) * l : 1);
    reset_nonfinite(c);
    {
        PhaseTimer timer(c, "streamed_upload");
        std::vector<cudaEvent_t> landed(static_cast<size_t>(C), nullptr);
        struct Events {
            std::vector<cudaEvent_t>& v;
            ~Events() {
                for (cudaEvent_t e : v)
                    if (e) cudaEventDestroy(e);
            }
        } guard{landed};
        SVDK_CUDA(cudaEventRecord(c->copy_ev, S));  // dA is ours on S (pool reuse)
        SVDK_CUDA(cudaStreamWaitEvent(c->copy_stream, c->copy_ev, 0));
        // Omega goes through the copy engine right after chunk 0 (both on the
        // copy stream; queued on the context stream it would wait behind every
        // chunk of A in the engine's FIFO), while the host joins its sampler.
        // Each chunk's copy is enqueued right before its compute: with a
        // pageable host buffer the enqueue packs the chunk through pinned
        // staging on this thread (HostUploader), which then overlaps the DMA
        // and compute of the chunks before it.
        HostUploader up(c, host);
        auto enqueue_copy = [&](int64_t k) {
            const int64_t r0 = k * rows, mk = std::min(rows, m - r0);
            up.copy2d(dA.p() + r0, lda * sizeof(double), host + r0, m * sizeof(double), mk * sizeof(double), n);
            if (k == 0) omega_upload(c, n, l, seed, Om.p(), c->copy_stream);
            SVDK_CUDA(cudaEventCreateWithFlags(&landed[k], cudaEventDisableTiming));
            SVDK_CUDA(cudaEventRecord(landed[k], c->copy_stream));
        };
        const bool trace = std::getenv("SVDK_STREAM_TRACE") != nullptr;
        std::vector<cudaEvent_t> tev;
        auto mark = [&](cudaStream_t st) {
            if (!trace) return;
            cudaEvent_t e;
            SVDK_CUDA(cudaEventCreate(&e));
            SVDK_CUDA(cudaEventRecord(e, st));
            tev.push_back(e);
        };
        mark(S);
        for (int64_t k = 0; k < C; ++k) {
            const int64_t r0 = k * rows, mk = std::min(rows, m - r0);
            double* Ak = dA.p() + r0;
            double* muk = mu_k.p() + k * n;
            enqueue_copy(k);
            SVDK_CUDA(cudaStreamWaitEvent(S, landed[k], 0));
            mark(S);
            column_sums(c, Ak, lda, mk, n, static_cast<double>(mk), muk);
            subtract_column_means(c, Ak, lda, mk, n, muk, Ak, lda);
            gemm(c, false, mk, l, n, Ak, lda, Om.p(), n, H.p() + r0, ldh, nullptr, true);  // H_k = A_k^c Omega
            if (with_z) {  // s_k and Z += A_k^c^T H_k
                column_sums(c, H.p() + r0, ldh, mk, l, 1.0, SH.p() + k * l);
                gemm(c, true, n, l, mk, Ak, lda, H.p() + r0, ldh, Z.p(), n, nullptr, false, 1.0, k > 0);
            }
            mark(S);
        }
        if (trace) {
            SVDK_CUDA(cudaStreamSynchronize(S));
            std::fprintf(stderr, "[stream trace] S events (ms from start, before/after each chunk):");
            for (size_t i = 1; i < tev.size(); ++i) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, tev[0], tev[i]);
                std::fprintf(stderr, " %.2f", ms);
            }
            std::fprintf(stderr, "\n");
            for (cudaEvent_t e : tev) cudaEventDestroy(e);
        }
    }
    const int64_t ldd = round_up(C, 2);
    DBuf d(c, static_cast<size_t>(ldd) * n), Wd(c, static_cast<size_t>(ldd) * l);
    if (ldd != C) fill(c, d.p(), ldd * n, 0.0);
    chunk_means_kernel<<<static_cast<unsigned>(ceil_div(n, 128)), 128, 0, S>>>(mu_k.p(), static_cast<int>(C), n,
                                                                               rows, m, mu.p(), d.p(), ldd);
    SVDK_CHECK_LAUNCH();
    gemm(c, false, ldd, l, n, d.p(), ldd, Om.p(), n, Wd.p(), ldd);  // row k = (Omega^T d_k)^T
    Om.reset();
    if (with_z) {  // Z += D^T E, E row k = s_k + cnt_k w_k
        DBuf E(c, static_cast<size_t>(ldd) * l);
        sketch_corr_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(ldd * l, 256), 4 * c->num_sms)), 256,
                             0, S>>>(SH.p(), Wd.p(), static_cast<int>(C), l, rows, m, ldd, E.p());
        SVDK_CHECK_LAUNCH();
        c->launches++;
        gemm(c, true, n, l, ldd, d.p(), ldd, E.p(), ldd, Z.p(), n, nullptr, false, 1.0, true);
    }
    {
        const dim3 gh(static_cast<unsigned>(std::min<int64_t>(ceil_div(m, 256), 2 * c->num_sms)),
                      static_cast<unsigned>(std::min<int64_t>(l, 256)));
        add_chunk_rows_kernel<<<gh, 256, 0, S>>>(H.p(), ldh, m, l, Wd.p(), ldd, rows, nullptr);
        SVDK_CHECK_LAUNCH();
        const dim3 ga(static_cast<unsigned>(std::min<int64_t>(ceil_div(m, 256), 2 * c->num_sms)),
                      static_cast<unsigned>(std::min<int64_t>(n, 256)));
        DBuf partial(c, static_cast<size_t>(ga.x) * ga.y + 1);
        add_chunk_rows_kernel<<<ga, 256, 0, S>>>(dA.p(), lda, m, n, d.p(), ldd, rows, partial.p());
        SVDK_CHECK_LAUNCH();
        sum_fixed_order_kernel<<<1, 32, 0, S>>>(partial.p(), static_cast<int>(ga.x * ga.y),
                                                partial.p() + static_cast<size_t>(ga.x) * ga.y);
        SVDK_CHECK_LAUNCH();
        c->launches += 4;
        d2h(c, total, partial.p() + static_cast<size_t>(ga.x) * ga.y, 1);
    }
    int64_t ldu, ldv;
    DBuf dU = alloc_mat(c, m, l, ldu), dV = alloc_mat(c, n, l, ldv), dS(c, std::max(l, n));
    const int64_t r = randomized_from_sketch(c, dA.p(), lda, m, n, l, q, std::move(H), ldh, dU.p(), ldu, dS.p(),
                                             dV.p(), ldv, nullptr, with_z ? Z.p() : nullptr);
    raise_if_nonfinite(c);
    download(c, basis, dV.p(), ldv, n, r);  // RowsAreExamples: basis = V
    std::vector<double> sv(r);
    download(c, sv.data(), dS.p(), r, r, 1);
    for (int64_t i = 0; i < r; ++i) eigenvalues[i] = sv[i] * sv[i];
    download(c, mean, mu.p(), n, n, 1);
    *rank = r;
    return true;
}

}  // namespace

bool fit_pca_streamed(Ctx* c, const double* host, int64_t m, int64_t n, int method, int64_t l, int64_t q,
                      uint64_t seed, double* basis, double* eigenvalues, double* total, double* mean,
                      int64_t* rank) {
    if (const char* e = std::getenv("SVDK_STREAM"))
        if (std::string(e) == "0") return false;
    if (method != SVDK_TRUNCATED && method != SVDK_RANDOMIZED) return false;
    if (m < n || n == 0 || has_comm(c)) return false;
    if (!c->copy_stream) {
        SVDK_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        SVDK_CUDA(cudaEventCreateWithFlags(&c->copy_ev, cudaEventDisableTiming));
    }
    if (method == SVDK_RANDOMIZED)
        return streamed_sketch_rows(c, host, m, n, l, q, seed, basis, eigenvalues, total, mean, rank);
    const int64_t nc = chunk_cols(m, n);
    if (nc <= 0 || nc >= n) return false;
    // truncated: column chunks under the block-column Gram
    validate_method(method, m, n, l, q, "fit_pca");
    const int64_t C = ceil_div(n, nc);
    cudaStream_t S = c->stream;
    int64_t lda;
    DBuf dA = alloc_mat(c, m, n, lda);
    DBuf mu(c, n), sq(c, C + 1), G(c, static_cast<size_t>(n) * n);
    reset_nonfinite(c);
    {
        PhaseTimer timer(c, "streamed_upload");
        std::vector<cudaEvent_t> landed(static_cast<size_t>(C), nullptr);
        struct Events {
            std::vector<cudaEvent_t>& v;
            ~Events() {
                for (cudaEvent_t e : v)
                    if (e) cudaEventDestroy(e);
            }
        } guard{landed};
        // the copy stream may only overwrite dA once it is ours on S (pool reuse)
        SVDK_CUDA(cudaEventRecord(c->copy_ev, S));
        SVDK_CUDA(cudaStreamWaitEvent(c->copy_stream, c->copy_ev, 0));
        HostUploader up(c, host);  // see streamed_sketch_rows: copy k is enqueued right before compute k
        for (int64_t k = 0; k < C; ++k) {
            const int64_t j0 = k * nc, cols = std::min(nc, n - j0), j1 = j0 + cols;
            double* Ak = dA.p() + j0 * lda;
            if (lda == m)
                up.copy2d(Ak, sizeof(double) * m * cols, host + j0 * m, sizeof(double) * m * cols,
                          sizeof(double) * m * cols, 1);
            else
                up.copy2d(Ak, lda * sizeof(double), host + j0 * m, m * sizeof(double), m * sizeof(double), cols);
            SVDK_CUDA(cudaEventCreateWithFlags(&landed[k], cudaEventDisableTiming));
            SVDK_CUDA(cudaEventRecord(landed[k], c->copy_stream));
            SVDK_CUDA(cudaStreamWaitEvent(S, landed[k], 0));
            // whole columns: mean, subtract and sum of squares exactly as for the full matrix
            column_sums(c, Ak, lda, m, cols, static_cast<double>(m), mu.p() + j0);
            subtract_column_means_sumsq(c, Ak, lda, m, cols, mu.p() + j0, Ak, lda, sq.p() + k);
            gemm(c, true, j1, cols, m, dA.p(), lda, Ak, lda, G.p() + j0 * n, n);  // upper block column G[0:j1, j0:j1]
        }
    }
    sum_fixed_order_kernel<<<1, 32, 0, S>>>(sq.p(), static_cast<int>(C), sq.p() + C);
    SVDK_CHECK_LAUNCH();
    c->launches++;
    d2h(c, total, sq.p() + C, 1);
    mirror_upper_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(n * n, 256), 4 * c->num_sms)), 256, 0,
                          S>>>(G.p(), n, n);
    SVDK_CHECK_LAUNCH();
    c->launches++;
    // the rest of the method on the centred, resident A
    int64_t ldu, ldv;
    DBuf dU = alloc_mat(c, m, n, ldu), dV = alloc_mat(c, n, n, ldv), dS(c, n);
    const int64_t r =
        truncated_from_gram(c, dA.p(), lda, m, n, std::move(G), dU.p(), ldu, dS.p(), dV.p(), ldv, nullptr);
    raise_if_nonfinite(c);
    download(c, basis, dV.p(), ldv, n, r);  // RowsAreExamples: basis = V
    std::vector<double> s(r);
    download(c, s.data(), dS.p(), r, r, 1);
    for (int64_t i = 0; i < r; ++i) eigenvalues[i] = s[i] * s[i];
    download(c, mean, mu.p(), n, n, 1);
    *rank = r;
    return true;
}

}  // namespace svdk
