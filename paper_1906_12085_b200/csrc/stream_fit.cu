// stream_fit.cu — fit_pca from a HOST buffer with the upload streamed under
// the first pass over A (reference pca.cpp:91-116 + svd_methods.cpp:121-170).
//
// svdk_fit_pca's plain path copies all of A to the GPU, then centres it, then
// runs the method: the PCIe copy (30 ms at c2, 1.2 s at c4) and the first pass
// over A (the Gram for truncated, H = A Omega for randomized) run back to back.
// Here A arrives in COLUMN chunks (contiguous in the column-major host buffer,
// so each is one full-speed DMA) on a copy stream, and the compute stream works
// on the chunks that have landed: a chunk holds whole columns, so it is centred
// exactly as the reference centres the matrix (column mean, then subtract,
// pca.cpp:37-53, fused with the chunk's sum of squares for the total variance),
// and then contributes its share of the first pass:
//   truncated:  G[0:j1, j0:j1] = A[:, 0:j1]^T A[:, j0:j1]  (the upper block
//               column; the upper triangle is mirrored at the end, as the
//               reference's gram computes i <= j and mirrors, kernels.cpp:80-97)
//   randomized: H += A[:, j0:j1] Omega[j0:j1, :]
// The rest of the method then runs on the resident, centred A.
#include <algorithm>
#include <cmath>
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

__global__ void sum_fixed_order_kernel(const double* partial, int count, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < count; ++i) s += partial[i];
        *out = s;
    }
}

// Columns per chunk (a multiple of 64, so chunks stay TMA-aligned): ~n/8 for
// the Gram (each block column of G is written once), ~n/4 for the sketch (every
// chunk re-reads and re-writes all of H, so fewer, longer-K chunks);
// 0 = do not stream (fewer than 2 chunks, or too little data to matter).
int64_t chunk_cols(int64_t m, int64_t n, int method) {
    if (const char* e = std::getenv("SVDK_STREAM_COLS")) {  // test / tuning override
        const int64_t v = std::atoll(e);
        return v <= 0 ? 0 : round_up(std::max<int64_t>(v, 64), 64);
    }
    if (8.0 * static_cast<double>(m) * static_cast<double>(n) < 64.0 * (1 << 20)) return 0;
    return round_up(std::max<int64_t>(ceil_div(n, method == SVDK_TRUNCATED ? 8 : 4), 64), 64);
}

}  // namespace

bool fit_pca_streamed(Ctx* c, const double* host, int64_t m, int64_t n, int method, int64_t l, int64_t q,
                      uint64_t seed, double* basis, double* eigenvalues, double* total, double* mean,
                      int64_t* rank) {
    if (const char* e = std::getenv("SVDK_STREAM"))
        if (std::string(e) == "0") return false;
    // Randomized: measured slower than upload-then-GEMM at c2 (169 / 164 ms with
    // 4 / 2 K-chunks of H += A_J Omega_J vs 161 ms): only the last chunk's GEMM
    // is saved while every chunk re-reads and re-writes H; opt in with
    // SVDK_STREAM=2 (kept for the parity tests and for other shapes).
    const char* mode = std::getenv("SVDK_STREAM");
    const bool sketch_ok = mode && std::string(mode) == "2";
    if (method != SVDK_TRUNCATED && !(method == SVDK_RANDOMIZED && sketch_ok)) return false;
    if (m < n || n == 0 || (c->nccl_comm && c->world > 1)) return false;
    const int64_t nc = chunk_cols(m, n, method);
    if (nc <= 0 || nc >= n) return false;
    validate_method(method, m, n, l, q, "fit_pca");
    const int64_t C = ceil_div(n, nc);
    const int64_t w = method_width(method, m, n, l, q);
    cudaStream_t S = c->stream;
    if (!c->copy_stream) {
        SVDK_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        SVDK_CUDA(cudaEventCreateWithFlags(&c->copy_ev, cudaEventDisableTiming));
    }
    int64_t lda;
    DBuf dA = alloc_mat(c, m, n, lda);
    DBuf mu(c, n), sq(c, C + 1);
    const int64_t ldh = round_up(m, 2);
    DBuf G, H, Om;
    if (method == SVDK_TRUNCATED) {
        G = DBuf(c, static_cast<size_t>(n) * n);
    } else {
        H = DBuf(c, static_cast<size_t>(ldh) * l);
        Om = DBuf(c, static_cast<size_t>(n) * l);
    }
    reset_nonfinite(c);
    {
        PhaseTimer timer(c, "streamed_upload");
        // every chunk's copy is enqueued first (one event each), so that the
        // copy engine never waits on the host (e.g. the Omega sampler below)
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
        for (int64_t k = 0; k < C; ++k) {
            const int64_t j0 = k * nc, cols = std::min(nc, n - j0);
            if (lda == m)
                SVDK_CUDA(cudaMemcpyAsync(dA.p() + j0 * lda, host + j0 * m, sizeof(double) * m * cols,
                                          cudaMemcpyHostToDevice, c->copy_stream));
            else
                SVDK_CUDA(cudaMemcpy2DAsync(dA.p() + j0 * lda, lda * sizeof(double), host + j0 * m,
                                            m * sizeof(double), m * sizeof(double), cols, cudaMemcpyHostToDevice,
                                            c->copy_stream));
            SVDK_CUDA(cudaEventCreateWithFlags(&landed[k], cudaEventDisableTiming));
            SVDK_CUDA(cudaEventRecord(landed[k], c->copy_stream));
        }
        // the reference sampler's Omega (prefetched on a host thread by the caller)
        if (method == SVDK_RANDOMIZED) omega_upload(c, n, l, seed, Om.p());
        for (int64_t k = 0; k < C; ++k) {
            const int64_t j0 = k * nc, cols = std::min(nc, n - j0), j1 = j0 + cols;
            double* Ak = dA.p() + j0 * lda;
            SVDK_CUDA(cudaStreamWaitEvent(S, landed[k], 0));
            // whole columns: mean, subtract and sum of squares exactly as for the full matrix
            column_sums(c, Ak, lda, m, cols, static_cast<double>(m), mu.p() + j0);
            subtract_column_means_sumsq(c, Ak, lda, m, cols, mu.p() + j0, Ak, lda, sq.p() + k);
            if (method == SVDK_TRUNCATED)  // upper block column G[0:j1, j0:j1]
                gemm(c, true, j1, cols, m, dA.p(), lda, Ak, lda, G.p() + j0 * n, n);
            else  // H += A[:, j0:j1] Omega[j0:j1, :]
                gemm(c, false, m, l, cols, Ak, lda, Om.p() + j0, n, H.p(), ldh, nullptr, true, 1.0, k > 0);
        }
    }
    sum_fixed_order_kernel<<<1, 32, 0, S>>>(sq.p(), static_cast<int>(C), sq.p() + C);
    SVDK_CHECK_LAUNCH();
    c->launches++;
    d2h(c, total, sq.p() + C, 1);
    if (method == SVDK_TRUNCATED) {
        mirror_upper_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(n * n, 256), 4 * c->num_sms)), 256, 0,
                              S>>>(G.p(), n, n);
        SVDK_CHECK_LAUNCH();
        c->launches++;
    } else {
        Om.reset();
    }
    // the rest of the method on the centred, resident A
    int64_t ldu, ldv;
    DBuf dU = alloc_mat(c, m, w, ldu), dV = alloc_mat(c, n, w, ldv), dS(c, std::max(w, n));
    int64_t r = 0;
    if (method == SVDK_TRUNCATED)
        r = truncated_from_gram(c, dA.p(), lda, m, n, std::move(G), dU.p(), ldu, dS.p(), dV.p(), ldv, nullptr);
    else
        r = randomized_from_sketch(c, dA.p(), lda, m, n, l, q, std::move(H), ldh, dU.p(), ldu, dS.p(), dV.p(),
                                   ldv, nullptr);
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
