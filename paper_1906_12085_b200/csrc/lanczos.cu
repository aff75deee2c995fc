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
// The GEMV pair is HBM-bound (4mn flop over 8mn bytes): a 4-CTA cluster
// streams each 64-row slab of A once from HBM (columns split over the CTAs);
// the slab's second use (A^T y) hits L2. Per-cluster column partials are
// reduced in fixed order. The per-step tail (alpha, CGS2, beta, breakdown
// restart) is decided on the device, so steps are enqueued back to back.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "svdk_methods.h"
#include "tma_util.h"

namespace svdk {
int64_t back_project(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* w,
                     const double* Vfull, int64_t ldvf, int64_t kcols, double* U, int64_t ldu,
                     double* sigma, double* V, int64_t ldv);

namespace {

// ---------------------------------------------------------------------------
// GEMV pair w = A^T (A q) in ONE read of A from HBM (default).
//
// A is cut into 64-row slabs; a cluster of CS CTAs (CS SMs) owns one slab at a
// time and CTA rank r of the cluster streams the slab's column range
// [r*ncta, (r+1)*ncta) as 64 x 32 TMA boxes (16 KB: 32 contiguous 512-byte
// runs). Each box is loaded twice: the first pass (y = A_slab q, evict_last)
// pulls it from HBM, the second (A_slab^T y, evict_first) re-reads it from L2.
// The CTAs of a cluster exchange their 64 partial y over distributed shared
// memory (one 512-byte cp.async.bulk push per peer, completing on the peer's
// mbarrier) and every CTA sums the CS partials in rank order, so y is
// bit-identical across the cluster. Pass 1 of slab i+1 runs before pass 2 of
// slab i, so the exchange has a slab of work to hide behind.
//
// Why this shape (tools/probes/stream_tma.cu, B200, 500000 x 2048, no math):
// one-pass TMA streaming of A reaches 7.2-7.3 TB/s for any box shape with
// >= 256-byte runs, but re-reading 32-row slabs of all 2048 columns from L2
// drops to 4.6 TB/s; 64-row boxes with the columns split over 4 CTAs keep the
// re-read at 6.9 TB/s (n = 2048) / 6.6 TB/s (n = 4096), and the L2 footprint
// between the two reads is nclusters x 64 x n x 8 B (39 MB at n = 2048).
//
// Warp roles per CTA: one producer thread issues the ring; consumer warp w owns
// ring stage w and takes tiles k = w, w + NCW, ... of the CTA's tile sequence
// (no shared-memory contention between warps). Lanes are rows (lane, lane+32).
// Pass 2 reduces each 32-column tile across lanes with a 31-shuffle butterfly
// (lane l ends with column l's sum). Per-cluster column partials go to
// partial[cluster][n] and are summed in fixed order by reduce_parts_kernel.
// Ring: GC_NST stages of 16 KB; tile k of the sequence lands in stage
// k % GC_NST and is consumed by warp k % GC_NCW. GC_NST must be a multiple of
// GC_NCW so a stage is always reused by the same warp, in order: a second warp
// waiting on the stage's next phase before the current one completes would
// see the parity of the already-completed phase and read a stale tile.
constexpr int GC_NCW = 6;                  // consumer warps (2 tiles in flight each)
constexpr int GC_NST = 2 * GC_NCW;         // ring stages
static_assert(GC_NST % GC_NCW == 0, "stage reuse must stay within one warp");
constexpr int GC_ROWS = 64, GC_COLS = 32;  // TMA box (rows x columns)
constexpr int GC_TILE = GC_ROWS * GC_COLS;
// y-exchange buffers: with one slab of lookahead a CTA writes slab i+1's
// partial while a lagging peer may still read slab i-2's; 4 buffers keep
// every write at least one completed wait behind the peer's last read.
constexpr int GC_YB = 4;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
}
// address of the same shared-memory object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_peer(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}

struct GcLayout {
    int ncta;  // columns per CTA (multiple of GC_COLS)
    size_t smem;
};
inline GcLayout gc_layout(int64_t n, int cs) {
    GcLayout L;
    L.ncta = static_cast<int>(ceil_div(ceil_div(n, cs), GC_COLS) * GC_COLS);
    L.smem = sizeof(double) * (static_cast<size_t>(GC_NST) * GC_TILE + 2 * L.ncta + 2 * GC_NCW * GC_ROWS +
                               GC_YB * cs * GC_ROWS) +
             (2 * GC_NST + GC_YB) * sizeof(uint64_t);
    return L;
}

template <int CS, bool LA>
__global__ void __launch_bounds__((GC_NCW + 1) * 32, 1)
    gemv_pair_cluster_kernel(const __grid_constant__ CUtensorMap mapA, int64_t m, int64_t n, int ncta,
                             const double* __restrict__ q, double* __restrict__ partial) {
    // declared (not computed) shared base: keeps every access below an LDS/STS
    // (a uintptr_t-aligned pointer compiles to generic LD/ST)
    extern __shared__ __align__(1024) double gc_smem[];
    double* ring = gc_smem;
    double* qs = ring + GC_NST * GC_TILE;         // ncta (zero beyond n)
    double* wacc = qs + ncta;                     // ncta
    double* ypart = wacc + ncta;                  // 2 x GC_NCW x 64: per-warp partial y (slab parity)
    double* ybuf = ypart + 2 * GC_NCW * GC_ROWS;  // GC_YB x CS x 64: cluster partials
    uint64_t* full = reinterpret_cast<uint64_t*>(ybuf + GC_YB * CS * GC_ROWS);
    uint64_t* empty = full + GC_NST;
    uint64_t* ybar = empty + GC_NST;              // GC_YB
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const int64_t col0 = static_cast<int64_t>(rank) * ncta;
    const int T = static_cast<int>(std::max<int64_t>(0, std::min<int64_t>(ncta, n - col0) + GC_COLS - 1) / GC_COLS);
    for (int j = tid; j < ncta; j += blockDim.x) {
        qs[j] = col0 + j < n ? q[col0 + j] : 0.0;
        wacc[j] = 0.0;
    }
    if (tid == 0) {
        for (int s = 0; s < GC_NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < GC_YB; ++s) mbar_init(&ybar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cluster_sync_all();  // peers' barriers are initialised before any remote arrive
    const int64_t nslabs = (m + GC_ROWS - 1) / GC_ROWS;
    const int64_t first = cluster_id_x(), stride = nclusters_x();
    const int64_t ns = nslabs > first ? (nslabs - first + stride - 1) / stride : 0;  // this cluster's slabs
    // Tile sequence (producer and consumers alike); tile k -> stage k % GC_NST,
    // consumed by warp k % GC_NCW. With lookahead (LA):
    //   P1(0), then for i = 0..ns-1: [P1(i+1)], P2(i)
    // so a slab's y exchange has a whole slab of work to hide behind;
    // without: P1(0), P2(0), P1(1), P2(1), ... (half the L2 residency).
    if (warp == GC_NCW) {  // ---------------- producer
        if (lane == 0 && T > 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
            const uint64_t keep = l2_policy_evict_last(), drop = l2_policy_evict_first();
            int64_t k = 0;
            auto issue = [&](int64_t i, bool second) {
                const int row0 = static_cast<int>((first + i * stride) * GC_ROWS);
                for (int t = 0; t < T; ++t, ++k) {
                    const int st = static_cast<int>(k % GC_NST);
                    const uint32_t use = static_cast<uint32_t>(k / GC_NST);
                    mbar_wait(&empty[st], (use & 1) ^ 1);
                    mbar_expect_tx(&full[st], GC_TILE * 8);
                    tma_load_2d_hint(ring + st * GC_TILE, &mapA, &full[st], row0,
                                     static_cast<int>(col0) + t * GC_COLS, second ? drop : keep);
                }
            };
            if (LA) {
                if (ns > 0) issue(0, false);
                for (int64_t i = 0; i < ns; ++i) {
                    if (i + 1 < ns) issue(i + 1, false);
                    issue(i, true);
                }
            } else {
                for (int64_t i = 0; i < ns; ++i) {
                    issue(i, false);
                    issue(i, true);
                }
            }
        }
    } else {  // ---------------- consumers
        int64_t kb = 0;  // sequence index of the segment's first tile
        // pass 1 of slab i: partial y over this CTA's columns -> every CTA's ybuf
        auto pass1 = [&](int64_t i) {
            double y0 = 0.0, y1 = 0.0;
            const int t0 = static_cast<int>(((warp - kb) % GC_NCW + GC_NCW) % GC_NCW);
            for (int t = t0; t < T; t += GC_NCW) {
                const int64_t k = kb + t;
                const int st = static_cast<int>(k % GC_NST);
                mbar_wait(&full[st], static_cast<uint32_t>(k / GC_NST) & 1);
                const double* tile = ring + st * GC_TILE;
                const double* qt = qs + t * GC_COLS;
                double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll 8
                for (int c = 0; c < GC_COLS; c += 2) {
                    const double2 qq = *reinterpret_cast<const double2*>(qt + c);
                    a0 = fma(tile[c * GC_ROWS + lane], qq.x, a0);
                    b0 = fma(tile[c * GC_ROWS + lane + 32], qq.x, b0);
                    a1 = fma(tile[(c + 1) * GC_ROWS + lane], qq.y, a1);
                    b1 = fma(tile[(c + 1) * GC_ROWS + lane + 32], qq.y, b1);
                }
                y0 += a0 + a1;
                y1 += b0 + b1;
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
            }
            kb += T;
            double* yp = ypart + (i & 1) * GC_NCW * GC_ROWS;
            yp[warp * GC_ROWS + lane] = y0;
            yp[warp * GC_ROWS + lane + 32] = y1;
            asm volatile("bar.sync 1, %0;" ::"r"(GC_NCW * 32) : "memory");
            if (warp == 0) {  // CTA partial -> slot `rank` of every CTA of the cluster
                double v0 = 0.0, v1 = 0.0;
#pragma unroll
                for (int w = 0; w < GC_NCW; ++w) {
                    v0 += yp[w * GC_ROWS + lane];
                    v1 += yp[w * GC_ROWS + lane + 32];
                }
                const int b = static_cast<int>(i % GC_YB);
                double* slot = ybuf + (b * CS + rank) * GC_ROWS;
                slot[lane] = v0;
                slot[lane + 32] = v1;
                // make the generic-proxy writes visible to the bulk-copy (async) proxy
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    // one 512-byte DSMEM push per peer, completing on the peer's ybar[b]
                    for (int p = 0; p < CS; ++p) {
                        if (p == static_cast<int>(rank)) continue;
                        asm volatile(
                            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes"
                            " [%0], [%1], %2, [%3];" ::"r"(map_peer(slot, p)),
                            "r"(smem_u32(slot)), "r"(GC_ROWS * 8), "r"(map_peer(&ybar[b], p))
                            : "memory");
                    }
                    // own arrival arms the phase for the CS-1 incoming partials
                    mbar_expect_tx(&ybar[b], (CS - 1) * GC_ROWS * 8);
                }
            }
        };
        if (LA && ns > 0) pass1(0);
        for (int64_t i = 0; i < ns; ++i) {
            // pass1's barrier also orders the previous slab's wacc updates
            // before this slab's (tile t of pass 2 moves between warps)
            if (!LA)
                pass1(i);
            else if (i + 1 < ns)
                pass1(i + 1);
            else
                asm volatile("bar.sync 1, %0;" ::"r"(GC_NCW * 32) : "memory");
            // y of slab i: the CS partials summed in rank order (identical in every CTA)
            const int b = static_cast<int>(i % GC_YB);
            mbar_wait(&ybar[b], static_cast<uint32_t>(i / GC_YB) & 1);
            double y0 = 0.0, y1 = 0.0;
#pragma unroll
            for (int p = 0; p < CS; ++p) {
                y0 += ybuf[(b * CS + p) * GC_ROWS + lane];
                y1 += ybuf[(b * CS + p) * GC_ROWS + lane + 32];
            }
            // pass 2 of slab i: w_j += sum_rows A[row, j] y_row over this warp's tiles
            const int t0 = static_cast<int>(((warp - kb) % GC_NCW + GC_NCW) % GC_NCW);
            for (int t = t0; t < T; t += GC_NCW) {
                const int64_t k = kb + t;
                const int st = static_cast<int>(k % GC_NST);
                mbar_wait(&full[st], static_cast<uint32_t>(k / GC_NST) & 1);
                const double* tile = ring + st * GC_TILE;
                double p[32];
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    p[c] = fma(tile[c * GC_ROWS + lane + 32], y1, tile[c * GC_ROWS + lane] * y0);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);  // tile consumed into registers
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    const bool upper = (lane & off) != 0;
#pragma unroll
                    for (int i2 = 0; i2 < off; ++i2) {
                        const double send = upper ? p[i2] : p[i2 + off];
                        const double keep = upper ? p[i2 + off] : p[i2];
                        p[i2] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                    }
                }
                wacc[t * GC_COLS + lane] += p[0];
            }
            kb += T;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(GC_NCW * 32) : "memory");
        double* out = partial + static_cast<int64_t>(first) * n + col0;
        for (int j = tid; j < ncta && col0 + j < n; j += GC_NCW * 32) out[j] = wacc[j];
    }
    __syncwarp();
    cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
}

// launch helper: grid = clusters x CS CTAs (one CTA per SM)
template <int CS, bool LA>
void launch_gemv_cluster(Ctx* c, const CUtensorMap& map, const double* A, int64_t lda, int64_t m, int64_t n,
                         const GcLayout& L, int nclusters, const double* q, double* partial) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(nclusters * CS));
    cfg.blockDim = dim3((GC_NCW + 1) * 32);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    (void)A;
    (void)lda;
    SVDK_CUDA(cudaLaunchKernelEx(&cfg, gemv_pair_cluster_kernel<CS, LA>, map, m, n, L.ncta, q, partial));
}

// Sets the kernel's shared-memory limit and returns how many CS-CTA clusters
// can be co-resident: clusters must sit inside one GPC, so on B200 only 33
// clusters of 4 (132 SMs) or 15 of 8 fit at once — launching floor(148/CS)
// would run the remainder as a second wave.
template <int CS, bool LA>
int prepare_gemv_cluster(const GcLayout& L, int num_sms) {
    ensure_smem_attr(reinterpret_cast<const void*>(gemv_pair_cluster_kernel<CS, LA>), L.smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(num_sms / CS * CS));
    cfg.blockDim = dim3((GC_NCW + 1) * 32);
    cfg.dynamicSmemBytes = L.smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int active = 0;
    SVDK_CUDA(cudaOccupancyMaxActiveClusters(&active, gemv_pair_cluster_kernel<CS, LA>, &cfg));
    return std::max(1, std::min(active, num_sms / CS));
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

// s + sum_{b < count} p[b * stride], added in index order (bit-identical to
// the plain loop) with 8 loads in flight instead of one
__device__ __forceinline__ double ordered_sum(double s, const double* p, int count, int64_t stride) {
    int b = 0;
    for (; b + 8 <= count; b += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + (b + u) * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; b < count; ++b) s += __ldcg(p + b * stride);
    return s;
}
// x - sum in the same order: x -= p[0], x -= p[stride], ...
__device__ __forceinline__ double ordered_sub(double x, const double* p, int count, int64_t stride) {
    int b = 0;
    for (; b + 8 <= count; b += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + (b + u) * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) x -= v[u];
    }
    for (; b < count; ++b) x -= __ldcg(p + b * stride);
    return x;
}

__global__ void reduce_parts_kernel(const double* partial, int parts, int64_t n, double* w) {
    const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    w[j] = ordered_sum(0.0, partial + j, parts, n);
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

// Last-CTA-done pattern: every CTA publishes its partial, fences, and bumps
// a counter; the CTA that sees the final count reduces the partials in index
// order (deterministic) and resets the counter for the next launch.
__device__ __forceinline__ bool last_cta_done(unsigned* counter, unsigned total) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        last = atomicAdd(counter, 1u) == total - 1;
        if (last) *counter = 0;
    }
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// w = sum of the GEMV's `parts` column partials (parts = 0: w is already
// summed, e.g. after the allreduce), then a_j = q^T w and
// w -= a_j q + b_{j-1} q_{j-1}. One thread per entry; the dot product is
// reduced per CTA and finished by the last CTA, which also applies the update.
__global__ void __launch_bounds__(256) reduce_alpha_kernel(const double* partial, int parts, int64_t n,
                                                            double* w, const double* q, const double* qprev,
                                                            const double* beta_prev, double* alpha_out,
                                                            double* dots, unsigned* counter, double* nrm0) {
    __shared__ double red[32];
    const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    double d = 0.0;
    if (j < n) {
        double s;
        if (parts > 0) {
            s = ordered_sum(0.0, partial + j, parts, n);
            w[j] = s;
        } else {
            s = w[j];
        }
        d = q[j] * s;
    }
    d = block_sum(d, red);
    if (threadIdx.x == 0) dots[blockIdx.x] = d;
    if (!last_cta_done(counter, gridDim.x)) return;
    double a = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) a += __ldcg(dots + b);
    const double bp = beta_prev ? *beta_prev : 0.0;
    double ss = 0.0;
    // one CTA walks all of w: 8 entries per thread in flight at a time (the
    // plain loop was a chain of dependent L2 round trips, ~16 us at n = 4096)
    constexpr int U = 8;
    for (int64_t i0 = threadIdx.x; i0 < n; i0 += U * static_cast<int64_t>(blockDim.x)) {
        double xw[U], xq[U], xp[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * static_cast<int64_t>(blockDim.x);
            xw[u] = i < n ? __ldcg(w + i) : 0.0;
            xq[u] = i < n ? q[i] : 0.0;
            xp[u] = (qprev && i < n) ? qprev[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * static_cast<int64_t>(blockDim.x);
            if (i < n) {
                double x = xw[u] - a * xq[u];
                if (qprev) x -= bp * xp[u];
                w[i] = x;
                ss = fma(x, x, ss);
            }
        }
    }
    ss = block_sum(ss, red);
    if (threadIdx.x == 0) {
        *alpha_out = a;
        *nrm0 = sqrt(ss);  // ||w|| before reorthogonalisation
    }
}

// h_k = Q[:, k]^T w for k < cols (one warp per column, 8 independent chains:
// Q_j is L2-resident and this is load-latency bound)
__global__ void __launch_bounds__(256) cgs_dot_kernel(const double* Q, int64_t ldq, int64_t n, int64_t cols,
                                                       const double* w, double* h, const double* skip) {
    if (skip && *skip != 0.0) return;  // second pass not needed this step
    const int64_t k = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (k >= cols) return;
    const double* qk = Q + k * ldq;
    double s[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) s[u] = 0.0;
    int64_t i = lane;
    for (; i + 7 * 32 < n; i += 8 * 32) {
        double x[8], y[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x[u] = __ldcg(qk + i + u * 32);
            y[u] = w[i + u * 32];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] = fma(x[u], y[u], s[u]);
    }
    for (; i < n; i += 32) s[0] = fma(qk[i], w[i], s[0]);
    double t = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) h[k] = t;
}

// w -= Q_cols h, then ||w||. CTA (rb, kc) sums columns [kc*kw, (kc+1)*kw) for
// rows [256 rb, 256 rb + 256) into part[kc][i]; the last CTA of a row block
// subtracts the kc partials in order and publishes the block's sum of squares;
// the last row block finishes ||w|| (fixed order throughout).
constexpr int CGS_ROWS = 256;
constexpr int CGS_MAXKC = 48;  // column chunks: ~a wave of CTAs at n = 2048
// Pass 1 (decide != nullptr) also applies "twice is enough" (Kahan-Parlett):
// if ||w1|| >= ||w0|| / sqrt(2) the projection removed only rounding-level
// components, w1 is orthogonal to Q_j to working precision, and pass 2 is
// skipped (its kernels see *skip != 0 and return; nrm[1] = nrm[0]). When it
// removed more (loss of orthogonality, or a true breakdown), pass 2 runs.
__global__ void __launch_bounds__(CGS_ROWS) cgs_update_norm_kernel(const double* Q, int64_t ldq, int64_t n,
                                                                   int64_t cols, int64_t kw, const double* h,
                                                                   double* w, double* part, double* sq,
                                                                   unsigned* counters, double* nrm_out,
                                                                   const double* nrm0, double* skip) {
    if (!nrm0 && skip && *skip != 0.0) return;  // pass 2, not needed this step
    __shared__ double hs[512];
    __shared__ double red[32];
    const int rb = blockIdx.x, kc = blockIdx.y, nkc = gridDim.y, nrb = gridDim.x;
    const int64_t i = static_cast<int64_t>(rb) * CGS_ROWS + threadIdx.x;
    const int64_t k0 = kc * kw, k1 = min(cols, k0 + kw);
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    for (int64_t kb = k0; kb < k1; kb += 512) {
        const int64_t ke = min(k1, kb + 512);
        __syncthreads();
        for (int64_t k = kb + threadIdx.x; k < ke; k += CGS_ROWS) hs[k - kb] = h[k];
        __syncthreads();
        if (i < n) {
            const double* qi = Q + i + kb * ldq;
            const int cnt = static_cast<int>(ke - kb);
            int k = 0;
            for (; k + 7 < cnt; k += 8) {
                double x[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = __ldcg(qi + (k + u) * ldq);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[u] = fma(x[u], hs[k + u], acc[u]);
            }
            for (; k < cnt; ++k) acc[0] = fma(qi[k * ldq], hs[k], acc[0]);
        }
    }
    if (i < n)
        part[kc * n + i] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    if (!last_cta_done(counters + rb, nkc)) return;
    double ss = 0.0;
    if (i < n) {
        const double x = ordered_sub(__ldcg(w + i), part + i, nkc, n);
        w[i] = x;
        ss = x * x;
    }
    ss = block_sum(ss, red);
    if (threadIdx.x == 0) sq[rb] = ss;
    if (!last_cta_done(counters + nrb, nrb)) return;
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int b = 0; b < nrb; ++b) t += __ldcg(sq + b);
        const double nw = sqrt(t);
        *nrm_out = nw;
        if (nrm0) {  // pass 1: decide whether pass 2 is needed
            const bool enough = nw >= 0.70710678118654752 * *nrm0;
            *skip = enough ? 1.0 : 0.0;
            if (enough) nrm_out[1] = nw;
        }
    }
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

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// End of Lanczos step j, decided on the device (no host round trip per step):
// nrm = {||w|| before, after} the second CGS pass, state = {gnorm, prev_beta,
// restart flag}. gnorm is the running Gershgorin bound on ||T||. Breakdown
// (an invariant subspace: the second reorthogonalisation pass removed more
// than half of w, or ||w|| <= 1e-14 ||T||) sets b_j = 0 and restarts with a
// fresh Gaussian vector (counter hash of (seed, j), identical on every rank),
// orthogonalised twice against Q_cols (CGS2) and normalised into q_{j+1} —
// by this same CTA: breakdowns are rare and Q_cols is read 4 times, so no
// grid-wide synchronisation is needed. Otherwise b_j = ||w|| and
// q_{j+1} = w / b_j.
__global__ void __launch_bounds__(1024) lanczos_finish_kernel(double* w, int64_t n, const double* nrm,
                                                              const double* alpha_j, double* beta_j,
                                                              double* state, double* qn, int last, uint64_t seed,
                                                              int64_t j, const double* Q, int64_t cols, double* h) {
    __shared__ int brk;
    __shared__ double red[32];
    const double n1 = nrm[0], n2 = nrm[1];
    const double gnorm = fmax(state[0], fabs(*alpha_j) + state[1] + n2);
    if (threadIdx.x == 0) brk = !last && (!(n2 > 0.5 * n1) || !(n2 > 1e-14 * gnorm));
    __syncthreads();
    if (threadIdx.x == 0) {
        state[0] = gnorm;
        *beta_j = brk ? 0.0 : n2;
        state[1] = brk ? 0.0 : n2;
    }
    if (last) return;
    if (!brk) {
        const double inv = 1.0 / n2;
        constexpr int U = 4;
        for (int64_t i0 = threadIdx.x; i0 < n; i0 += U * static_cast<int64_t>(blockDim.x)) {
            double x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = i0 + u * static_cast<int64_t>(blockDim.x);
                x[u] = i < n ? __ldcg(w + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = i0 + u * static_cast<int64_t>(blockDim.x);
                if (i < n) qn[i] = x[u] * inv;
            }
        }
        return;
    }
    const uint64_t key = splitmix64(seed ^ (0x9e3779b97f4a7c15ull * static_cast<uint64_t>(j + 1)));
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t h1 = splitmix64(key + 2 * static_cast<uint64_t>(i));
        const uint64_t h2 = splitmix64(key + 2 * static_cast<uint64_t>(i) + 1);
        const double u1 = static_cast<double>((h1 >> 11) + 1) * 0x1.0p-53;
        const double u2 = static_cast<double>(h2 >> 11) * 0x1.0p-53;
        w[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int pass = 0; pass < 2; ++pass) {
        for (int64_t k = warp; k < cols; k += nw) {
            double s = 0.0;
            for (int64_t i = lane; i < n; i += 32) s = fma(Q[k * n + i], w[i], s);
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) h[k] = s;
        }
        __syncthreads();
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            double s = 0.0;
            for (int64_t k = 0; k < cols; ++k) s = fma(Q[k * n + i], h[k], s);
            w[i] -= s;
        }
        __syncthreads();
    }
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(w[i], w[i], s);
    const double inv = 1.0 / sqrt(block_sum(s, red));
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) qn[i] = w[i] * inv;
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

// w = A^T (A q) in the form picked for (A, m, n): "cluster" (default) reads A
// once from HBM with the column range of a 64-row slab split over a CS-CTA
// cluster; "twopass" streams A twice along its columns (fallback for shapes
// TMA cannot address). SVDK_GEMV=cluster|twopass and SVDK_GEMV_CS=1|2|4|8
// override (development knobs; the tests sweep them).
GemvPair::GemvPair(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n)
    : c_(c), A_(A), lda_(lda), m_(m), n_(n) {
    const char* gv_env = std::getenv("SVDK_GEMV");
    int smem_optin = 0;
    SVDK_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    const bool shape_ok = m > 0 && (lda % 2 == 0) && m < (int64_t(1) << 31) && n < (int64_t(1) << 31) &&
                          (reinterpret_cast<uintptr_t>(A) % 16 == 0);
    cluster_ = shape_ok && !(gv_env && std::string(gv_env) == "twopass");
    const char* cs_env = std::getenv("SVDK_GEMV_CS");
    if (const char* e = std::getenv("SVDK_GEMV_LA")) la_ = std::atoi(e) != 0;
    // Cluster size: the smallest whose slab set stays L2-resident between a
    // tile's two reads — co-resident clusters x (1 + lookahead) slabs x 64 rows
    // x n x 8 B <= 72 MiB (of the 126 MB L2) — among those whose shared memory fits.
    auto prepare = [&](int cs, const GcLayout& gl) {
        switch (cs * 2 + (la_ ? 1 : 0)) {
            case 2: return prepare_gemv_cluster<1, false>(gl, c->num_sms);
            case 3: return prepare_gemv_cluster<1, true>(gl, c->num_sms);
            case 4: return prepare_gemv_cluster<2, false>(gl, c->num_sms);
            case 5: return prepare_gemv_cluster<2, true>(gl, c->num_sms);
            case 8: return prepare_gemv_cluster<4, false>(gl, c->num_sms);
            case 9: return prepare_gemv_cluster<4, true>(gl, c->num_sms);
            case 16: return prepare_gemv_cluster<8, false>(gl, c->num_sms);
            default: return prepare_gemv_cluster<8, true>(gl, c->num_sms);
        }
    };
    bool chosen = false;
    for (int cs : {1, 2, 4, 8}) {
        if (!cluster_) break;
        if (cs_env && std::atoi(cs_env) != cs) continue;
        const GcLayout gl = gc_layout(n, cs);
        if (gl.smem > static_cast<size_t>(smem_optin)) continue;
        const int active = prepare(cs, gl);
        const double footprint = static_cast<double>(active) * (la_ ? 2 : 1) * GC_ROWS * n * 8;
        cs_ = cs;
        nclusters_ = active;
        ncta_ = gl.ncta;
        smem_ = gl.smem;
        chosen = true;
        if (cs_env || footprint <= 72.0 * (1 << 20)) break;
    }
    cluster_ = cluster_ && chosen;
    if (cluster_) {
        map_ = tensor_map_2d(A, m, n, lda, GC_ROWS, GC_COLS, CU_TENSOR_MAP_SWIZZLE_NONE);
        partial_ = DBuf(c, static_cast<size_t>(nclusters_) * std::max<int64_t>(n, 1));
    } else {
        const int64_t row_blocks = ceil_div(std::max<int64_t>(m, 1), GN_THREADS * GN_ROWS);
        chunks_ = std::min<int64_t>(std::max<int64_t>(1, ceil_div(2 * c->num_sms, row_blocks)),
                                    std::max<int64_t>(1, n / 16));
        yv_ = DBuf(c, static_cast<size_t>(std::max<int64_t>(m, 1)) * chunks_);
    }
}

void GemvPair::run(const double* q, double* w, bool reduce) {
    Ctx* c = c_;
    if (n_ == 0) return;
    if (m_ == 0) {
        fill(c, w, n_, 0.0);
        return;
    }
    {
        PhaseTimer timer(c, "gemv_pair", 4.0 * m_ * n_, 8.0 * m_ * n_);
        if (cluster_) {
            const GcLayout gl{ncta_, smem_};
            double* pp = partial_.p();
            switch (cs_ * 2 + (la_ ? 1 : 0)) {
                case 2: launch_gemv_cluster<1, false>(c, map_, A_, lda_, m_, n_, gl, nclusters_, q, pp); break;
                case 3: launch_gemv_cluster<1, true>(c, map_, A_, lda_, m_, n_, gl, nclusters_, q, pp); break;
                case 4: launch_gemv_cluster<2, false>(c, map_, A_, lda_, m_, n_, gl, nclusters_, q, pp); break;
                case 5: launch_gemv_cluster<2, true>(c, map_, A_, lda_, m_, n_, gl, nclusters_, q, pp); break;
                case 8: launch_gemv_cluster<4, false>(c, map_, A_, lda_, m_, n_, gl, nclusters_, q, pp); break;
                case 9: launch_gemv_cluster<4, true>(c, map_, A_, lda_, m_, n_, gl, nclusters_, q, pp); break;
                case 16: launch_gemv_cluster<8, false>(c, map_, A_, lda_, m_, n_, gl, nclusters_, q, pp); break;
                default: launch_gemv_cluster<8, true>(c, map_, A_, lda_, m_, n_, gl, nclusters_, q, pp); break;
            }
            c->launches++;
        } else {
            const int64_t row_blocks = ceil_div(m_, GN_THREADS * GN_ROWS);
            gemv_n_kernel<<<dim3(static_cast<unsigned>(row_blocks), static_cast<unsigned>(chunks_)), GN_THREADS,
                            0, c->stream>>>(A_, lda_, m_, n_, q, yv_.p());
            SVDK_CHECK_LAUNCH();
            if (chunks_ > 1) {
                sum_chunks_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(m_, 256), 4 * c->num_sms)),
                                    256, 0, c->stream>>>(yv_.p(), m_, static_cast<int>(chunks_));
                SVDK_CHECK_LAUNCH();
                c->launches++;
            }
            gemv_t_kernel<<<static_cast<unsigned>(n_), GT_THREADS, 0, c->stream>>>(A_, lda_, m_, yv_.p(), w);
            c->launches += 2;
        }
        SVDK_CHECK_LAUNCH();
    }
    if (cluster_ && reduce) {
        reduce_parts_kernel<<<static_cast<unsigned>(ceil_div(n_, 256)), 256, 0, c->stream>>>(
            partial_.p(), nclusters_, n_, w);
        SVDK_CHECK_LAUNCH();
        c->launches++;
    }
}

bool tridiag_eig(Ctx* c, const double* alpha, const double* beta, int64_t k, double* w, double* S, int64_t lds);

int64_t lanczos_svd(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t steps,
                    uint64_t seed, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                    const RowComm* comm) {
    if (steps <= 0 || steps > n) steps = n;
    GemvPair gemv(c, A, lda, m, n);
    DBuf Q(c, static_cast<size_t>(n) * (steps + 1)), w(c, n), h(c, steps + 1), scal(c, 2 * steps + 8);
    double* alpha = scal.p();
    double* beta = scal.p() + steps;
    double* nrm = scal.p() + 2 * steps;    // [0] after CGS pass 1, [1] after pass 2
    double* state = scal.p() + 2 * steps + 2;  // gnorm, prev_beta, (unused), ||w0||, skip pass 2
    fill(c, state, 5, 0.0);
    // step-tail workspaces: per-CTA partials and last-CTA counters (zeroed once;
    // every kernel resets the counters it used)
    const int64_t nb256 = ceil_div(n, 256);
    DBuf part(c, static_cast<size_t>(CGS_MAXKC) * n), red(c, static_cast<size_t>(nb256) + 8), cntbuf(c, nb256 + 8);
    unsigned* cnt = reinterpret_cast<unsigned*>(cntbuf.p());
    SVDK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(double) * (nb256 + 8), c->stream));
    // q_0 = g / ||g|| with g from the reference sampler
    omega_upload(c, n, 1, seed, w.p());
    norm_kernel<<<1, 1024, 0, c->stream>>>(w.p(), n, nrm);
    scale_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c->stream>>>(w.p(), n, nrm, Q.p());
    SVDK_CHECK_LAUNCH();
    c->launches += 2;
    // Every step is enqueued without a host round trip: the breakdown decision
    // and the restart run on the device (lanczos_finish_kernel).
    for (int64_t j = 0; j < steps; ++j) {
        const double* qj = Q.p() + j * n;
        // w = A^T A q_j (GEMV partials reduced in reduce_alpha unless an
        // allreduce over row shards has to sit between the two)
        gemv.run(qj, w.p(), /*reduce=*/comm != nullptr);
        if (comm) comm->allreduce(w.p(), static_cast<size_t>(n));
        const int parts = comm ? 0 : gemv.parts();
        reduce_alpha_kernel<<<static_cast<unsigned>(nb256), 256, 0, c->stream>>>(
            gemv.partials(), parts, n, w.p(), qj, j > 0 ? Q.p() + (j - 1) * n : nullptr,
            j > 0 ? beta + (j - 1) : nullptr, alpha + j, red.p(), cnt, state + 3);
        SVDK_CHECK_LAUNCH();
        const int64_t cols = j + 1;
        const int64_t nkc = std::min<int64_t>(CGS_MAXKC, ceil_div(cols, 32));
        const int64_t kw = ceil_div(cols, nkc);
        for (int pass = 0; pass < 2; ++pass) {
            double* skip = state + 4;  // set by pass 1, read by pass 2
            cgs_dot_kernel<<<static_cast<unsigned>(ceil_div(cols * 32, 256)), 256, 0, c->stream>>>(
                Q.p(), n, n, cols, w.p(), h.p(), pass == 1 ? skip : nullptr);
            SVDK_CHECK_LAUNCH();
            cgs_update_norm_kernel<<<dim3(static_cast<unsigned>(nb256), static_cast<unsigned>(nkc)), CGS_ROWS,
                                     0, c->stream>>>(Q.p(), n, n, cols, kw, h.p(), w.p(), part.p(), red.p(),
                                                     cnt + 1, nrm + pass, pass == 0 ? state + 3 : nullptr, skip);
            SVDK_CHECK_LAUNCH();
        }
        const bool last = j + 1 == steps;
        double* qn = last ? nullptr : Q.p() + (j + 1) * n;
        lanczos_finish_kernel<<<1, 1024, 0, c->stream>>>(w.p(), n, nrm, alpha + j, beta + j, state, qn,
                                                         last ? 1 : 0, seed, j, Q.p(), cols, h.p());
        SVDK_CHECK_LAUNCH();
        c->launches += 6;
    }
    // Ritz pairs: eig(T) by the O(k^2) tridiagonal solver (bisection + twisted
    // factorisation, tridiag.cu); T with unresolved clusters (e.g. the repeated
    // Ritz values after a breakdown restart) goes to the dense Jacobi solver.
    const int64_t lds = round_up(steps, 2);
    DBuf theta(c, steps), S(c, static_cast<size_t>(lds) * steps);
    const char* tri_env = std::getenv("SVDK_LANCZOS_TRIDIAG");
    const bool try_tri = !(tri_env && std::atoi(tri_env) == 0);
    if (!try_tri || !tridiag_eig(c, alpha, beta, steps, theta.p(), S.p(), lds)) {
        PhaseTimer timer(c, "tridiag_dense");
        DBuf T(c, static_cast<size_t>(steps) * steps);
        tridiag_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(steps * steps, 256), 1024)), 256,
                         0, c->stream>>>(alpha, beta, steps, T.p());
        SVDK_CHECK_LAUNCH();
        c->launches++;
        eig_sym(c, T.p(), steps, steps, 30, theta.p(), S.p(), lds);
    }
    DBuf Vr(c, static_cast<size_t>(n) * steps);
    gemm(c, false, n, steps, steps, Q.p(), n, S.p(), lds, Vr.p(), n);
    Q.reset();
    return back_project(c, A, lda, m, n, theta.p(), Vr.p(), n, steps, U, ldu, sigma, V, ldv);
}

}  // namespace svdk
