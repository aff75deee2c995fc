// lanczos.cu — Lanczos on A^T A with full reorthogonalisation (NEW method:
// the reference has block Krylov only, svd_methods.cpp:172-196, and lists
// Lanczos as a non-goal; BASELINE configs c3/c5 ask for it). Parity oracle:
// the reference truncated_svd (Gram + Jacobi) on the same A.
//
//   q_0 = g / ||g||, g = gaussian_matrix(n, 1, seed)  (reference sampler)
//   for j < steps:
//     w   = A^T (A q_j)           fused one-pass GEMV pair  [+ allreduce n]
//     a_j = q_j^T w ; w -= a_j q_j + b_{j-1} q_{j-1}
//     w  -= Q_j (Q_j^T w)  twice  (CGS2 full reorthogonalisation)
//     b_j = ||w|| ; q_{j+1} = w / b_j   (random restart on breakdown)
//   T = tridiag(a, b) -> Jacobi eig_sym -> Ritz V = Q_L S -> sigma, U = A V / sigma
//
// The GEMV pair is HBM-bound (4mn flop over 8mn bytes): each CTA streams its
// share of 32-row slabs of A once from HBM; the slab's second use (A^T y)
// hits L2. Per-CTA column partials are reduced in fixed order.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "svdk_methods.h"
#include "tma_util.h"

namespace svdk {
void gaussian_fill(int64_t rows, int64_t cols, uint64_t seed, double* out);
int64_t back_project(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* w,
                     const double* Vfull, int64_t ldvf, int64_t kcols, double* U, int64_t ldu,
                     double* sigma, double* V, int64_t ldv);

namespace {

constexpr int GV_WARPS = 8;
constexpr int GV_THREADS = GV_WARPS * 32;
constexpr int GV_U = 16;     // independent 256-byte column loads in flight per lane
constexpr int GV_CTAS_PER_SM = 2;  // two CTAs per SM drift out of phase, so one
                                   // streams HBM (phase 1) while the other
                                   // re-reads its slab from L2 (phase 2)

// partial[b][j] = sum over this CTA's 32-row slabs of A_slab^T (A_slab q).
// Lane l of every warp owns row l of the slab (coalesced 256 B per column).
//  phase 1: y = A_slab q — warp w sums columns w, w+8, ... with GV_U loads
//           in flight per lane, then the 16 partial y are combined in smem;
//  phase 2: for blocks of 32 columns a lane keeps 32 partial products in
//           registers, and a 31-shuffle butterfly transposes and reduces them
//           so lane l ends with the full column sum of column l.
// The slab's second read (phase 2) hits L2: 296 CTAs x 32 rows x n x 8 B.
template <int GV_WARPS, int CPS>
__global__ void __launch_bounds__(GV_WARPS * 32, CPS)
    gemv_pair_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                     const double* __restrict__ q, double* __restrict__ partial) {
    constexpr int GV_THREADS = GV_WARPS * 32;
    extern __shared__ double sm[];
    double* qs = sm;            // n
    double* wacc = sm + n;      // n
    double* ypart = wacc + n;   // GV_WARPS x 32
    __shared__ double y[32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int64_t j = tid; j < n; j += GV_THREADS) {
        qs[j] = q[j];
        wacc[j] = 0.0;
    }
    __syncthreads();
    const int64_t nslabs = (m + 31) / 32;
    for (int64_t s = blockIdx.x; s < nslabs; s += gridDim.x) {
        const int64_t row = s * 32 + lane;
        const bool in = row < m;
        const double* a = A + (in ? row : 0);
        // ---- phase 1
        double acc[GV_U];
#pragma unroll
        for (int u = 0; u < GV_U; ++u) acc[u] = 0.0;
        int64_t j = warp;
        for (; j + (GV_U - 1) * GV_WARPS < n; j += GV_U * GV_WARPS) {
            double x[GV_U];
#pragma unroll
            for (int u = 0; u < GV_U; ++u) x[u] = in ? __ldg(a + (j + u * GV_WARPS) * lda) : 0.0;
#pragma unroll
            for (int u = 0; u < GV_U; ++u) acc[u] = fma(x[u], qs[j + u * GV_WARPS], acc[u]);
        }
        for (; j < n; j += GV_WARPS) acc[0] = fma(in ? a[j * lda] : 0.0, qs[j], acc[0]);
        double t = 0.0;
#pragma unroll
        for (int u = 0; u < GV_U; ++u) t += acc[u];
        ypart[warp * 32 + lane] = t;
        __syncthreads();
        if (warp == 0) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < GV_WARPS; ++w) v += ypart[w * 32 + lane];
            y[lane] = v;
        }
        __syncthreads();
        // ---- phase 2: 32-column blocks, warp w takes blocks w, w+GV_WARPS, ...
        const double yl = y[lane];
        for (int64_t c0 = warp * 32; c0 < n; c0 += GV_WARPS * 32) {
            double p[32];
#pragma unroll
            for (int c = 0; c < 32; ++c)
                p[c] = (in && c0 + c < n) ? a[(c0 + c) * lda] * yl : 0.0;
            // butterfly transpose-reduce: after the step with offset `off`,
            // lane l holds partial sums for the columns whose index agrees
            // with l in the bits above `off`
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                const bool upper = (lane & off) != 0;
#pragma unroll
                for (int i = 0; i < off; ++i) {
                    const double send = upper ? p[i] : p[i + off];
                    const double keep = upper ? p[i + off] : p[i];
                    p[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                }
            }
            // lane l now holds the sum of column c0 + l
            if (c0 + lane < n) wacc[c0 + lane] += p[0];
        }
        // ypart/y are rewritten next slab only after the first barrier above
    }
    __syncthreads();
    for (int64_t j = tid; j < n; j += GV_THREADS) partial[blockIdx.x * n + j] = wacc[j];
}

// Single-read GEMV pair streamed by TMA (default when n <= 2048):
//   w_partial[cta] = sum over the CTA's 32-row slabs of A_slab^T (A_slab q).
// One CTA per SM; one producer thread walks the CTA's slabs and issues, per
// slab, the T = ceil(n/64) column tiles (32 rows x 64 cols = 16 KB, one TMA
// box each) TWICE — the first pass (y = A_slab q) pulls them from HBM, the
// second (A_slab^T y) re-reads them from L2: 148 slabs x 32 rows x n x 8 B
// = 78 MB at n = 2048 stay resident. Consumer warp w owns ring stage w and
// takes tiles k = w, w + NCW, ... of the CTA's tile sequence, so the ring is
// NCW x 16 KB of loads in flight per SM with no shared-memory contention
// between warps. Per tile, lanes are rows: pass 1 is 64 conflict-free LDS +
// FMA per lane; pass 2 multiplies by y_lane and reduces each 32-column group
// across lanes with a 31-shuffle butterfly (lane l ends with column l's sum).
// The two passes of a slab are separated by one consumer-only named barrier
// (y complete); partial y are double-buffered by slab parity.
constexpr int GT_NCW = 8;                 // consumer warps = ring stages
constexpr int GT_ROWS = 32, GT_COLS = 64; // TMA box
constexpr int GT_TILE = GT_ROWS * GT_COLS;

__global__ void __launch_bounds__((GT_NCW + 1) * 32, 1)
    gemv_pair_tma_kernel(const __grid_constant__ CUtensorMap mapA, int64_t m, int64_t n,
                         const double* __restrict__ q, double* __restrict__ partial) {
    extern __shared__ uint8_t gt_raw[];
    double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(gt_raw) + 127) & ~uintptr_t(127));
    const int T = static_cast<int>((n + GT_COLS - 1) / GT_COLS);
    const int npad = T * GT_COLS;
    double* qs = ring + GT_NCW * GT_TILE;   // npad (zero beyond n)
    double* wacc = qs + npad;               // npad
    double* ypart = wacc + npad;            // 2 x GT_NCW x 32
    uint64_t* full = reinterpret_cast<uint64_t*>(ypart + 2 * GT_NCW * 32);
    uint64_t* empty = full + GT_NCW;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int j = tid; j < npad; j += blockDim.x) {
        qs[j] = j < n ? q[j] : 0.0;
        wacc[j] = 0.0;
    }
    if (tid == 0) {
        for (int s = 0; s < GT_NCW; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t nslabs = (m + GT_ROWS - 1) / GT_ROWS;
    if (warp == GT_NCW) {  // ---------------- producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
            // first read: keep the tile in L2 for the second; second: drop it
            const uint64_t keep = l2_policy_evict_last(), drop = l2_policy_evict_first();
            int64_t k = 0;
            for (int64_t sl = blockIdx.x; sl < nslabs; sl += gridDim.x) {
                const int row0 = static_cast<int>(sl * GT_ROWS);
                for (int pass = 0; pass < 2; ++pass)
                    for (int t = 0; t < T; ++t, ++k) {
                        const int st = static_cast<int>(k % GT_NCW);
                        const uint32_t use = static_cast<uint32_t>(k / GT_NCW);
                        mbar_wait(&empty[st], (use & 1) ^ 1);
                        mbar_expect_tx(&full[st], GT_TILE * 8);
                        tma_load_2d_hint(ring + st * GT_TILE, &mapA, &full[st], row0, t * GT_COLS,
                                         pass == 0 ? keep : drop);
                    }
            }
        }
        return;
    }
    // ---------------- consumers
    double* tile = ring + warp * GT_TILE;  // this warp's stage
    uint32_t uses = 0;                     // completed uses of the stage
    int64_t base = 0;                      // CTA tile index of the slab's first tile
    int par = 0;
    for (int64_t sl = blockIdx.x; sl < nslabs; sl += gridDim.x, base += 2 * T, par ^= 1) {
        // pass 1: y_lane = sum_j A[row, j] q_j over this warp's tiles
        double yacc = 0.0;
        int t0 = static_cast<int>(((warp - base) % GT_NCW + GT_NCW) % GT_NCW);
        for (int t = t0; t < T; t += GT_NCW) {
            mbar_wait(&full[warp], uses & 1);
            const double* qt = qs + t * GT_COLS;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll 16
            for (int c = 0; c < GT_COLS; c += 2) {
                a0 = fma(tile[c * GT_ROWS + lane], qt[c], a0);
                a1 = fma(tile[(c + 1) * GT_ROWS + lane], qt[c + 1], a1);
            }
            yacc += a0 + a1;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[warp]);
            ++uses;
        }
        double* yp = ypart + par * GT_NCW * 32;
        yp[warp * 32 + lane] = yacc;
        asm volatile("bar.sync 1, %0;" ::"r"(GT_NCW * 32) : "memory");
        double y = 0.0;
#pragma unroll
        for (int w = 0; w < GT_NCW; ++w) y += yp[w * 32 + lane];
        // pass 2: w_j += sum_rows A[row, j] y_row over this warp's tiles
        t0 = static_cast<int>(((warp - base - T) % GT_NCW + GT_NCW) % GT_NCW);
        for (int t = t0; t < T; t += GT_NCW) {
            mbar_wait(&full[warp], uses & 1);
#pragma unroll
            for (int g = 0; g < GT_COLS / 32; ++g) {
                double p[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) p[c] = tile[(g * 32 + c) * GT_ROWS + lane] * y;
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    const bool upper = (lane & off) != 0;
#pragma unroll
                    for (int i = 0; i < off; ++i) {
                        const double send = upper ? p[i] : p[i + off];
                        const double keep = upper ? p[i + off] : p[i];
                        p[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                    }
                }
                wacc[t * GT_COLS + g * 32 + lane] += p[0];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[warp]);
            ++uses;
        }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(GT_NCW * 32) : "memory");
    for (int64_t j = tid; j < n; j += GT_NCW * 32) partial[blockIdx.x * n + j] = wacc[j];
}

size_t gemv_tma_smem(int64_t n) {
    const int64_t npad = ceil_div(n, GT_COLS) * GT_COLS;
    return 128 + sizeof(double) * (GT_NCW * GT_TILE + 2 * npad + 2 * GT_NCW * 32) + 2 * GT_NCW * 8;
}

// Two-pass streaming form of w = A^T (A q): both passes read A along
// its columns in long contiguous runs (DRAM-friendly), y (m doubles) lives in
// L2 between them, and no cross-CTA reduction is needed.
constexpr int GN_THREADS = 256, GN_ROWS = 4;  // rows per thread in y = A q
constexpr int GT_THREADS = 256;

// y_c[r] = sum_{j in chunk c} A[r, j] q[j]; CTA (b, c) owns rows
// [b R, (b+1) R), R = 256 * 4 (thread t rows t, t+256, ...: 256 B runs per
// warp, 8 KB per CTA) and column chunk c (gridDim.y chunks when m is short).
__global__ void __launch_bounds__(GN_THREADS)
    gemv_n_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                  const double* __restrict__ q, double* __restrict__ y) {
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * GN_THREADS * GN_ROWS + threadIdx.x;
    const int64_t cw = (n + gridDim.y - 1) / gridDim.y;
    const int64_t jb = blockIdx.y * cw, je = min(n, jb + cw);
    y += static_cast<int64_t>(blockIdx.y) * m;
    double acc[GN_ROWS];
    bool in[GN_ROWS];
#pragma unroll
    for (int u = 0; u < GN_ROWS; ++u) {
        acc[u] = 0.0;
        in[u] = r0 + u * GN_THREADS < m;
    }
    int64_t j = jb;
    for (; j + 1 < je; j += 2) {
        const double q0 = __ldg(q + j), q1 = __ldg(q + j + 1);
        const double* a0 = A + j * lda + r0;
        const double* a1 = a0 + lda;
        double x0[GN_ROWS], x1[GN_ROWS];
#pragma unroll
        for (int u = 0; u < GN_ROWS; ++u) {
            x0[u] = in[u] ? __ldcs(a0 + u * GN_THREADS) : 0.0;
            x1[u] = in[u] ? __ldcs(a1 + u * GN_THREADS) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < GN_ROWS; ++u) acc[u] = fma(x1[u], q1, fma(x0[u], q0, acc[u]));
    }
    if (j < je) {
        const double qj = __ldg(q + j);
#pragma unroll
        for (int u = 0; u < GN_ROWS; ++u)
            if (in[u]) acc[u] = fma(__ldcs(A + j * lda + r0 + u * GN_THREADS), qj, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < GN_ROWS; ++u)
        if (in[u]) y[r0 + u * GN_THREADS] = acc[u];
}

// y[r] = sum_c y_c[r] in chunk order (deterministic)
__global__ void sum_chunks_kernel(double* y, int64_t m, int chunks) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < m;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = y[r];
        for (int c = 1; c < chunks; ++c) s += y[c * m + r];
        y[r] = s;
    }
}

// w[j] = sum_i A[i, j] y[i]: one CTA per column, a contiguous m-run.
__global__ void __launch_bounds__(GT_THREADS)
    gemv_t_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                  const double* __restrict__ y, double* __restrict__ w) {
    __shared__ double red[GT_THREADS / 32];
    const double* a = A + static_cast<int64_t>(blockIdx.x) * lda;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t i = threadIdx.x;
    for (; i + 3 * GT_THREADS < m; i += 4 * GT_THREADS) {
        s0 = fma(__ldcs(a + i), __ldg(y + i), s0);
        s1 = fma(__ldcs(a + i + GT_THREADS), __ldg(y + i + GT_THREADS), s1);
        s2 = fma(__ldcs(a + i + 2 * GT_THREADS), __ldg(y + i + 2 * GT_THREADS), s2);
        s3 = fma(__ldcs(a + i + 3 * GT_THREADS), __ldg(y + i + 3 * GT_THREADS), s3);
    }
    for (; i < m; i += GT_THREADS) s0 = fma(__ldcs(a + i), __ldg(y + i), s0);
    double s = (s0 + s1) + (s2 + s3);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < GT_THREADS / 32; ++k) t += red[k];
        w[blockIdx.x] = t;
    }
}

__global__ void reduce_parts_kernel(const double* partial, int parts, int64_t n, double* w) {
    const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int b = 0; b < parts; ++b) s += partial[b * n + j];
    w[j] = s;
}

__device__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < (blockDim.x >> 5); ++i) t += red[i];
    return t;
}

// a_j = q^T w ; w -= a_j q + b_prev q_prev   (single CTA)
__global__ void alpha_kernel(double* w, const double* q, const double* qprev, int64_t n,
                             const double* beta_prev, double* alpha_out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(q[i], w[i], s);
    const double a = block_sum(s, red);
    const double b = beta_prev ? *beta_prev : 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double x = w[i] - a * q[i];
        if (qprev) x -= b * qprev[i];
        w[i] = x;
    }
    if (threadIdx.x == 0) *alpha_out = a;
}

// h_k = Q[:, k]^T w for k < cols (one warp per column)
__global__ void cgs_dot_kernel(const double* Q, int64_t ldq, int64_t n, int64_t cols,
                               const double* w, double* h) {
    const int64_t k = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (k >= cols) return;
    const double* qk = Q + k * ldq;
    double s = 0.0;
    for (int64_t i = lane; i < n; i += 32) s = fma(qk[i], w[i], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) h[k] = s;
}

// w_i -= sum_k Q[i,k] h_k (thread per row, coalesced over i)
__global__ void cgs_update_kernel(const double* Q, int64_t ldq, int64_t n, int64_t cols,
                                  const double* h, double* w) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double s0 = 0.0, s1 = 0.0;
    int64_t k = 0;
    for (; k + 1 < cols; k += 2) {
        s0 = fma(Q[i + k * ldq], h[k], s0);
        s1 = fma(Q[i + (k + 1) * ldq], h[k + 1], s1);
    }
    if (k < cols) s0 = fma(Q[i + k * ldq], h[k], s0);
    w[i] -= s0 + s1;
}

__global__ void norm_kernel(const double* w, int64_t n, double* out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(w[i], w[i], s);
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) *out = sqrt(t);
}

__global__ void scale_kernel(const double* w, int64_t n, const double* nrm, double* out) {
    const double inv = 1.0 / *nrm;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = w[i] * inv;
}

// Dense tridiagonal T (k x k) from alpha, beta.
__global__ void tridiag_kernel(const double* alpha, const double* beta, int64_t k, double* T) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < k * k;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / k, i = e - j * k;
        double v = 0.0;
        if (i == j)
            v = alpha[i];
        else if (i == j + 1)
            v = beta[j];
        else if (j == i + 1)
            v = beta[i];
        T[e] = v;
    }
}

}  // namespace

int64_t lanczos_svd(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t steps,
                    uint64_t seed, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                    const RowComm* comm) {
    if (steps <= 0 || steps > n) steps = n;
    // fused-GEMV geometry (development knob SVDK_GEMV_CFG = warps x CTAs/SM)
    int gv_warps = GV_WARPS, gv_cps = GV_CTAS_PER_SM;
    if (const char* e = std::getenv("SVDK_GEMV_CFG")) std::sscanf(e, "%dx%d", &gv_warps, &gv_cps);
    auto gv_kernel = gemv_pair_kernel<GV_WARPS, GV_CTAS_PER_SM>;
    if (gv_warps == 16 && gv_cps == 1) gv_kernel = gemv_pair_kernel<16, 1>;
    else if (gv_warps == 8 && gv_cps == 1) gv_kernel = gemv_pair_kernel<8, 1>;
    else if (gv_warps == 32 && gv_cps == 1) gv_kernel = gemv_pair_kernel<32, 1>;
    else if (gv_warps == 4 && gv_cps == 2) gv_kernel = gemv_pair_kernel<4, 2>;
    else { gv_warps = GV_WARPS; gv_cps = GV_CTAS_PER_SM; }
    const int parts = gv_cps * c->num_sms;
    const size_t gv_smem = (2 * n + gv_warps * 32) * sizeof(double);
    if (gv_smem > 200 * 1024) fail(SVDK_E_PARAM, "lanczos_svd: n too large for the fused GEMV");
    SVDK_CUDA(cudaFuncSetAttribute(gv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(gv_smem)));
    DBuf Q(c, static_cast<size_t>(n) * (steps + 1)), w(c, n), partial(c, static_cast<size_t>(parts) * n),
        h(c, steps + 1), scal(c, 2 * steps + 8);
    // GEMV-pair form: "fused" keeps a 32-row slab in L2 between A q and
    // A^T y (one HBM read, short DRAM runs); "two-pass" streams A twice along
    // its columns. SVDK_GEMV=fused|twopass overrides the default.
    const char* gv_env = std::getenv("SVDK_GEMV");
    const size_t tma_smem = gemv_tma_smem(n);
    const bool tma_ok = tma_smem <= 220 * 1024 && n <= 2048 && (lda % 2 == 0) &&
                        (reinterpret_cast<uintptr_t>(A) % 16 == 0);
    const std::string gv_mode = gv_env ? std::string(gv_env) : (tma_ok ? "tma" : "twopass");
    const bool use_tma = gv_mode == "tma" && tma_ok;
    const bool two_pass = !use_tma && gv_mode != "fused";
    CUtensorMap mapA{};
    if (use_tma) {
        mapA = tensor_map_2d(A, m, n, lda, GT_ROWS, GT_COLS, CU_TENSOR_MAP_SWIZZLE_NONE);
        SVDK_CUDA(cudaFuncSetAttribute(gemv_pair_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(tma_smem)));
    }
    const int64_t row_blocks = ceil_div(std::max<int64_t>(m, 1), GN_THREADS * GN_ROWS);
    const int64_t chunks = std::min<int64_t>(std::max<int64_t>(1, ceil_div(2 * c->num_sms, row_blocks)),
                                             std::max<int64_t>(1, n / 16));
    DBuf yv(c, static_cast<size_t>(std::max<int64_t>(m, 1)) * chunks);
    double* alpha = scal.p();
    double* beta = scal.p() + steps;
    double* nrm = scal.p() + 2 * steps;  // [0] after pass 1, [1] after pass 2
    // q_0 = g / ||g|| with g from the reference sampler
    omega_upload(c, n, 1, seed, w.p());
    norm_kernel<<<1, 1024, 0, c->stream>>>(w.p(), n, nrm);
    scale_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c->stream>>>(w.p(), n, nrm, Q.p());
    SVDK_CHECK_LAUNCH();
    c->launches += 2;
    double gnorm = 0.0;  // running Gershgorin bound on ||T||
    std::vector<double> hb(2);
    double prev_beta = 0.0;
    for (int64_t j = 0; j < steps; ++j) {
        const double* qj = Q.p() + j * n;
        if (two_pass) {
            PhaseTimer timer(c, "gemv_pair", 4.0 * m * n, 8.0 * m * n);
            gemv_n_kernel<<<dim3(static_cast<unsigned>(row_blocks), static_cast<unsigned>(chunks)),
                            GN_THREADS, 0, c->stream>>>(A, lda, m, n, qj, yv.p());
            SVDK_CHECK_LAUNCH();
            if (chunks > 1) {
                sum_chunks_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(m, 256), 4 * c->num_sms)),
                                    256, 0, c->stream>>>(yv.p(), m, static_cast<int>(chunks));
                SVDK_CHECK_LAUNCH();
            }
            gemv_t_kernel<<<static_cast<unsigned>(n), GT_THREADS, 0, c->stream>>>(A, lda, m, yv.p(),
                                                                                  w.p());
            SVDK_CHECK_LAUNCH();
        } else {
            {
                PhaseTimer timer(c, "gemv_pair", 4.0 * m * n, 8.0 * m * n);
                if (use_tma)
                    gemv_pair_tma_kernel<<<c->num_sms, (GT_NCW + 1) * 32, tma_smem, c->stream>>>(
                        mapA, m, n, qj, partial.p());
                else
                    gv_kernel<<<parts, gv_warps * 32, gv_smem, c->stream>>>(A, lda, m, n, qj,
                                                                            partial.p());
                SVDK_CHECK_LAUNCH();
            }
            reduce_parts_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c->stream>>>(
                partial.p(), use_tma ? c->num_sms : parts, n, w.p());
            SVDK_CHECK_LAUNCH();
        }
        if (comm) comm->allreduce(w.p(), static_cast<size_t>(n));
        alpha_kernel<<<1, 1024, 0, c->stream>>>(w.p(), qj, j > 0 ? Q.p() + (j - 1) * n : nullptr, n,
                                                j > 0 ? beta + (j - 1) : nullptr, alpha + j);
        SVDK_CHECK_LAUNCH();
        const int64_t cols = j + 1;
        for (int pass = 0; pass < 2; ++pass) {
            cgs_dot_kernel<<<static_cast<unsigned>(ceil_div(cols * 32, 256)), 256, 0, c->stream>>>(
                Q.p(), n, n, cols, w.p(), h.p());
            SVDK_CHECK_LAUNCH();
            cgs_update_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c->stream>>>(
                Q.p(), n, n, cols, h.p(), w.p());
            SVDK_CHECK_LAUNCH();
            norm_kernel<<<1, 1024, 0, c->stream>>>(w.p(), n, nrm + pass);
            SVDK_CHECK_LAUNCH();
        }
        c->launches += 9;
        double ab[3];
        SVDK_CUDA(cudaMemcpyAsync(hb.data(), nrm, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                  c->stream));
        SVDK_CUDA(cudaMemcpyAsync(ab, alpha + j, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        SVDK_CUDA(cudaStreamSynchronize(c->stream));
        const double n1 = hb[0], n2 = hb[1];
        gnorm = std::max(gnorm, std::fabs(ab[0]) + prev_beta + n2);
        if (j + 1 == steps) {
            SVDK_CUDA(cudaMemcpyAsync(beta + j, nrm + 1, sizeof(double), cudaMemcpyDeviceToDevice,
                                      c->stream));
            break;
        }
        double* qn = Q.p() + (j + 1) * n;
        const bool breakdown = !(n2 > 0.5 * n1) || !(n2 > 1e-14 * gnorm);
        if (!breakdown) {
            SVDK_CUDA(cudaMemcpyAsync(beta + j, nrm + 1, sizeof(double), cudaMemcpyDeviceToDevice,
                                      c->stream));
            scale_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c->stream>>>(
                w.p(), n, nrm + 1, qn);
            SVDK_CHECK_LAUNCH();
            c->launches++;
            prev_beta = n2;
        } else {
            // invariant subspace found: b_j = 0, restart with a random vector
            // orthogonalised (twice) against Q_j (replicated on every rank)
            const double zero = 0.0;
            h2d(c, beta + j, &zero, 1);
            std::vector<double> g(n);
            gaussian_fill(n, 1, seed ^ (0x9e3779b97f4a7c15ull * static_cast<uint64_t>(j + 1)),
                          g.data());
            h2d(c, w.p(), g.data(), n);
            for (int pass = 0; pass < 2; ++pass) {
                cgs_dot_kernel<<<static_cast<unsigned>(ceil_div(cols * 32, 256)), 256, 0,
                                 c->stream>>>(Q.p(), n, n, cols, w.p(), h.p());
                cgs_update_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c->stream>>>(
                    Q.p(), n, n, cols, h.p(), w.p());
            }
            norm_kernel<<<1, 1024, 0, c->stream>>>(w.p(), n, nrm);
            scale_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c->stream>>>(
                w.p(), n, nrm, qn);
            SVDK_CHECK_LAUNCH();
            c->launches += 6;
            prev_beta = 0.0;
        }
    }
    // Ritz pairs: eig(T), V = Q_L S
    DBuf T(c, static_cast<size_t>(steps) * steps), theta(c, steps), S(c, static_cast<size_t>(steps) * steps);
    tridiag_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(steps * steps, 256), 1024)), 256,
                     0, c->stream>>>(alpha, beta, steps, T.p());
    SVDK_CHECK_LAUNCH();
    c->launches++;
    eig_sym(c, T.p(), steps, steps, 30, theta.p(), S.p(), steps);
    DBuf Vr(c, static_cast<size_t>(n) * steps);
    gemm(c, false, n, steps, steps, Q.p(), n, S.p(), steps, Vr.p(), n);
    Q.reset();
    return back_project(c, A, lda, m, n, theta.p(), Vr.p(), n, steps, U, ldu, sigma, V, ldv);
}

}  // namespace svdk
