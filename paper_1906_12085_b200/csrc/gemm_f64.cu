// gemm_f64.cu — FP64 tensor-core GEMM / SYRK engine for sm_100a.
//
// Replaces the reference's scalar loop nests
//   gram                    kernels.cpp:80-97   (SYRK, upper tiles, exact mirror)
//   matmul_transposed_left  kernels.cpp:47-67   (TN, long-K split-K)
//   matmul                  kernels.cpp:14-45   (NN, + column-scale epilogue and
//                                                non-finite flag, :39-43)
//
// Hardware mapping (B200 / sm_100a):
//  * FP64 math runs on the DMMA pipe: mma.sync.m8n8k4.f64 lowers to
//    DMMA.8x8x4 (tcgen05 has no f64 kind). Measured pipe peak 37.0 TFLOP/s
//    vs 33.8 for DFMA (profiles/fp64_peaks.json).
//  * Operands stream HBM/L2 -> SMEM by TMA (cp.async.bulk.tensor, 128B
//    swizzle) into a 6-stage mbarrier ring filled by one producer warp;
//    eight consumer warps each own a 64x32 slice of the 128x128 CTA tile
//    (64 FP64 accumulators per thread in registers).
//  * Persistent grid: one CTA per SM walks (tile, k-split) work units in a
//    static round-robin, so concurrent CTAs share the same k-range of A in
//    L2. Split-K partials are reduced in a fixed order (deterministic; no
//    floating-point atomics), and SYRK writes each mirror pair from one value
//    so G is exactly symmetric like the reference.
//
// Shared-memory fragment layout and bank conflicts: with 128B swizzle a
// K-major tile holds element (c, k) at byte c*128 + (((k>>1) ^ (c&7))<<4) +
// (k&1)*8. The m8n8k4 fragment of a lane is (row = lane>>2, k = lane&3); we
// map MMA row r to tile row perm8(r) = 2*(r&3) + (r>>2) so the four rows a
// half-warp touches fall in distinct 32B bank groups (conflict-free LDS.64).
// The M-major tile (NN's A operand) uses the analogous map within 16 rows.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <utility>
#include <vector>

#include "svdk_internal.h"
#include "tma_util.h"

namespace svdk {
namespace {

constexpr int BM = 128, BN = 128, BK = 16;
constexpr int STAGES = 6;
constexpr int CWARPS = 8;                        // consumer warps (2 warpgroups)
constexpr int PWARPS = 4;                        // producer warpgroup (1 thread issues TMA)
constexpr int THREADS = (CWARPS + PWARPS) * 32;
constexpr int TILE_BYTES = BM * BK * 8;          // 16 KiB per operand per stage
constexpr int TILE_ELEMS = BM * BN;              // partial tile size (doubles)
constexpr int SMEM_BYTES = STAGES * 2 * TILE_BYTES + 1024 + 2 * STAGES * 8;

enum Kind : int { KIND_SYRK = 0, KIND_TN = 1, KIND_NN = 2 };
#ifdef SVDK_GEMM_NO_FAST_EPILOGUE  // bisection switch (development)
constexpr bool kFastEpilogue = false;
#else
constexpr bool kFastEpilogue = true;
#endif

struct Params {
    int kind;
    int a_mmajor;  // A operand is M-contiguous (NN)
    int64_t M, N, K;
    int tiles_m, tiles_n, n_tiles;
    int splits;
    int64_t k_per_split;
    int units;
    double* C;
    int64_t ldc;
    double* partial;
    const double* col_scale;
    int* flag;
    double alpha;  // out = alpha * (op(A) B) [+ C_old when beta_one]
    int beta_one;
    int b_upper;   // B is upper triangular: tile (., col0) only needs k < col0 + BN
    int a_tma3;    // M-major A via one 3-D box per stage (M % 16 == 0) instead of 8 2-D boxes
    // SYRK work line (see build_syrk_line): unit u = (tile, k0, k1) triples, the contiguous unit
    // range of every CTA and of every tile. Null: the uniform tiles x splits grid.
    const long long* utab;
    const long long* cfirst;
    const long long* tfirst;
    const long long* clist;  // CTA b runs the units clist[cfirst[b]] .. clist[cfirst[b + 1] - 1]
};

// 3-D box: (m_lo 16, k 16, m_hi 8) lands as m_lo*8 + k*128 + m_hi*2048 bytes,
// the same swizzled layout the eight 2-D 16x16 boxes produce.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// MMA row r (0..7) -> row within an 8-row K-major group.
__host__ __device__ __forceinline__ int perm8(int r) { return ((r & 3) << 1) | (r >> 2); }
// MMA row r of m-tile parity p -> row within a 16-row M-major group.
__host__ __device__ __forceinline__ int map16(int p, int r) {
    return (r & 1) + (((r >> 1) & 1) << 3) + ((r >> 2) << 1) + (p << 2);
}

struct Unit {
    int64_t row0, col0, k0, k1;
    bool diag;
};

__device__ __forceinline__ Unit decode(const Params& p, int u) {
    Unit w;
    if (p.utab) {  // SYRK work line: explicit (tile, k0, k1)
        const long long* e = p.utab + 3 * static_cast<size_t>(u);
        const int t = static_cast<int>(e[0]);
        int tj = static_cast<int>((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
        while ((tj + 1) * (tj + 2) / 2 <= t) ++tj;
        while (tj * (tj + 1) / 2 > t) --tj;
        const int ti = t - tj * (tj + 1) / 2;
        w.row0 = static_cast<int64_t>(ti) * BM;
        w.col0 = static_cast<int64_t>(tj) * BN;
        w.diag = ti == tj;
        w.k0 = e[1];
        w.k1 = e[2];
        return w;
    }
    const int split = u / p.n_tiles;
    const int t = u - split * p.n_tiles;
    int ti, tj;
    if (p.kind == KIND_SYRK) {
        // upper-triangular enumeration, column by column: t -> (ti <= tj)
        tj = static_cast<int>((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
        while ((tj + 1) * (tj + 2) / 2 <= t) ++tj;
        while (tj * (tj + 1) / 2 > t) --tj;
        ti = t - tj * (tj + 1) / 2;
    } else if (p.b_upper) {
        // triangular B: tile cost grows with tj, so walk column-major (all row
        // tiles of column 0, then column 1, ...): the round-robin CTA schedule
        // then gives every CTA an even mix of cheap and expensive tiles
        tj = t / p.tiles_m;
        ti = t - tj * p.tiles_m;
    } else {
        ti = t / p.tiles_n;
        tj = t - ti * p.tiles_n;
    }
    w.row0 = static_cast<int64_t>(ti) * BM;
    w.col0 = static_cast<int64_t>(tj) * BN;
    w.diag = (p.kind == KIND_SYRK) && (ti == tj);
    w.k0 = static_cast<int64_t>(split) * p.k_per_split;
    w.k1 = min(p.K, w.k0 + p.k_per_split);
    if (p.b_upper) w.k1 = min(w.k1, w.col0 + BN);
    if (w.k1 < w.k0) w.k1 = w.k0;
    return w;
}

// (idx, tid) of a thread-linear accumulator slot -> tile-local (row, col).
__device__ __forceinline__ void slot_coord(int a_mmajor, int idx, int tid, int& r, int& c) {
    const int warp = tid >> 5, lane = tid & 31;
    const int wm = warp >> 2, wn = warp & 3;
    const int t = idx >> 3, tn = (idx >> 1) & 3, i = idx & 1;
    const int lr = lane >> 2;
    r = wm * 64 + (a_mmajor ? 16 * (t >> 1) + map16(t & 1, lr) : t * 8 + perm8(lr));
    c = wn * 32 + tn * 8 + perm8(2 * (lane & 3) + i);
}

// The same for a diagonal SYRK tile of the work line, where consumer warp w
// holds the 8-row groups w and 15 - w against the column groups on or above
// the diagonal (17 of the tile's 136 upper 8 x 8 blocks per warp): slot
// (which, n, i) = acc[4 which + n / 4][n % 4][i].
__device__ __forceinline__ void slot_coord_diag(int idx, int tid, int& r, int& c) {
    const int warp = tid >> 5, lane = tid & 31;
    const int which = idx >> 5, n = (idx >> 1) & 15, i = idx & 1;
    r = (which ? 15 - warp : warp) * 8 + perm8(lane >> 2);
    c = n * 8 + perm8(2 * (lane & 3) + i);
}

__device__ __forceinline__ void store_out(const Params& p, int64_t row, int64_t col, double v) {
    if (row >= p.M || col >= p.N) return;
    if (p.kind == KIND_SYRK) {
        if (row > col) return;  // one value per mirror pair -> exact symmetry
        if (p.alpha != 1.0) v *= p.alpha;
        if (p.beta_one) v += p.C[row + col * p.ldc];
        p.C[row + col * p.ldc] = v;
        p.C[col + row * p.ldc] = v;
        return;
    }
    if (p.flag && !isfinite(v)) atomicOr(p.flag, 1);
    if (p.col_scale) v *= p.col_scale[col];
    if (p.alpha != 1.0) v *= p.alpha;
    if (p.beta_one) v += p.C[row + col * p.ldc];
    p.C[row + col * p.ldc] = v;
}

// The k loop of a diagonal SYRK tile for consumer warp W (compile-time, so the
// block selection below costs no branches and the operand loads are hoisted
// like in the main loop): row groups W and 15 - W against the column groups on
// or above the diagonal, 16 - W and W + 1 blocks = 17 DMMAs per k4-step for
// every warp (the four SM sub-partitions stay balanced); both operands come
// from the A stage. acc[4 which + n / 4][n % 4] = block (row group, n).
template <int W>
__device__ __forceinline__ void diag_unit(double (&acc)[8][4][2], const uint8_t* smA, uint64_t* full,
                                          uint64_t* empty, int& stage, uint32_t& phase, int64_t k0, int64_t k1,
                                          const uint32_t (&koff)[4], int lane) {
    constexpr int RB1 = W, RB2 = 15 - W, NMIN = RB1 < RB2 ? RB1 : RB2;
    for (int64_t k = k0; k < k1; k += BK) {
        mbar_wait(&full[stage], phase);
        const uint8_t* st = smA + stage * TILE_BYTES;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const double a1 = *reinterpret_cast<const double*>(st + RB1 * 1024 + koff[s]);
            const double a2 = *reinterpret_cast<const double*>(st + RB2 * 1024 + koff[s]);
            double bf[16];
#pragma unroll
            for (int n = NMIN; n < 16; ++n) bf[n] = *reinterpret_cast<const double*>(st + n * 1024 + koff[s]);
#pragma unroll
            for (int n = NMIN; n < 16; ++n) {
                if (n >= RB1) dmma(acc[n >> 2][n & 3][0], acc[n >> 2][n & 3][1], a1, bf[n]);
                if (n >= RB2) dmma(acc[4 + (n >> 2)][n & 3][0], acc[4 + (n >> 2)][n & 3][1], a2, bf[n]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
        }
    }
}

// TAB: the SYRK unit tables (its own instantiation, so the plain TN / NN kernels carry none of that code).
template <bool AMM, bool TAB = false>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                const Params p) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128B swizzle. Kept as a generic pointer:
    // the operand reads compile to generic LD (not LDS). Deriving `smem` from
    // the declared array instead (LDS operand reads, SVDK_GEMM_LDS) was 1%
    // faster alone but, combined with the direct-store epilogue below,
    // corrupted whole 8 x 32 accumulator groups in ~0.04% of 128 x 128 tiles
    // of 2^20 x 1024 x 1024 GEMMs (bitwise check vs cuBLAS on exactly
    // representable operands, tools/parity/gen_check2.py); this form: 0
    // mismatches in 48 such GEMMs and 35.6 TF/s (DESIGN 3.1).
#ifdef SVDK_GEMM_LDS  // development switch
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
#else
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
#endif
    uint8_t* smA = smem;
    uint8_t* smB = smem + STAGES * TILE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * STAGES * TILE_BYTES);
    uint64_t* empty = full + STAGES;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CWARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp >= CWARPS) {
        // ---------------- TMA producer warpgroup ----------------
        // Hand registers to the consumers: 1 producer + 2 consumer warps per
        // SM sub-partition fit 40 + 2 x 232 registers per lane.
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
        if (warp == CWARPS && lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA))
                         : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB))
                         : "memory");
            int stage = 0;
            uint32_t phase = 0;
            constexpr bool tab = TAB;
            const int u_begin = tab ? static_cast<int>(p.cfirst[blockIdx.x]) : static_cast<int>(blockIdx.x);
            const int u_end = tab ? static_cast<int>(p.cfirst[blockIdx.x + 1]) : p.units;
            const int u_step = tab ? 1 : static_cast<int>(gridDim.x);
            for (int j = u_begin; j < u_end; j += u_step) {
                const int u = tab ? static_cast<int>(p.clist[j]) : j;
                const Unit w = decode(p, u);
                for (int64_t k = w.k0; k < w.k1; k += BK) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], w.diag ? TILE_BYTES : 2 * TILE_BYTES);
                    uint8_t* da = smA + stage * TILE_BYTES;
                    if (AMM && p.a_tma3) {
                        tma_load_3d(da, &mapA, &full[stage], 0, static_cast<int>(k),
                                    static_cast<int>(w.row0 >> 4));
                    } else if (AMM) {
#pragma unroll
                        for (int b = 0; b < BM / 16; ++b)
                            tma_load_2d(da + b * 2048, &mapA, &full[stage],
                                        static_cast<int>(w.row0 + 16 * b), static_cast<int>(k));
                    } else {
                        tma_load_2d(da, &mapA, &full[stage], static_cast<int>(k),
                                    static_cast<int>(w.row0));
                    }
                    if (!w.diag)
                        tma_load_2d(smB + stage * TILE_BYTES, &mapB, &full[stage],
                                    static_cast<int>(k), static_cast<int>(w.col0));
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    const int wm = warp >> 2, wn = warp & 3;
    const int lr = lane >> 2, kq = lane & 3;
    const int p8 = perm8(lr);
    // K-major fragment offsets (bytes) for the 4 k4-steps of a BK=16 stage.
    uint32_t koff[4];
#pragma unroll
    for (int s = 0; s < 4; ++s)
        koff[s] = p8 * 128 + ((((2 * s + (kq >> 1)) ^ p8)) << 4) + ((kq & 1) << 3);
    // M-major fragment offsets for the two 8-row halves of a 16-row group.
    uint32_t moff[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int mlo = map16(h, lr);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int k = 4 * s + kq;
            moff[h][s] = k * 128 + ((((mlo >> 1) ^ (k & 7))) << 4) + ((mlo & 1) << 3);
        }
    }
    const uint32_t a_row_base = AMM ? wm * 4 * 2048 : wm * 64 * 128;
    const uint32_t b_row_base = wn * 32 * 128;

    double acc[8][4][2];
    int stage = 0;
    uint32_t phase = 0;
    constexpr bool tab = TAB;
    const int u_begin = tab ? static_cast<int>(p.cfirst[blockIdx.x]) : static_cast<int>(blockIdx.x);
    const int u_end = tab ? static_cast<int>(p.cfirst[blockIdx.x + 1]) : p.units;
    const int u_step = tab ? 1 : static_cast<int>(gridDim.x);
    for (int j = u_begin; j < u_end; j += u_step) {
        const int u = tab ? static_cast<int>(p.clist[j]) : j;
        const Unit w = decode(p, u);
#pragma unroll
        for (int t = 0; t < 8; ++t)
#pragma unroll
            for (int n = 0; n < 4; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;

        if (tab && w.diag) {
            // Diagonal tile of the SYRK work line: only the 136 upper 8 x 8 blocks
            // (diag_unit, one branch-free instantiation per consumer warp).
            switch (warp) {
                case 0: diag_unit<0>(acc, smA, full, empty, stage, phase, w.k0, w.k1, koff, lane); break;
                case 1: diag_unit<1>(acc, smA, full, empty, stage, phase, w.k0, w.k1, koff, lane); break;
                case 2: diag_unit<2>(acc, smA, full, empty, stage, phase, w.k0, w.k1, koff, lane); break;
                case 3: diag_unit<3>(acc, smA, full, empty, stage, phase, w.k0, w.k1, koff, lane); break;
                case 4: diag_unit<4>(acc, smA, full, empty, stage, phase, w.k0, w.k1, koff, lane); break;
                case 5: diag_unit<5>(acc, smA, full, empty, stage, phase, w.k0, w.k1, koff, lane); break;
                case 6: diag_unit<6>(acc, smA, full, empty, stage, phase, w.k0, w.k1, koff, lane); break;
                default: diag_unit<7>(acc, smA, full, empty, stage, phase, w.k0, w.k1, koff, lane); break;
            }
        } else
        for (int64_t k = w.k0; k < w.k1; k += BK) {
            mbar_wait(&full[stage], phase);
            const uint8_t* sa = smA + stage * TILE_BYTES + a_row_base;
            const uint8_t* sb = (w.diag ? smA : smB) + stage * TILE_BYTES + b_row_base;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                double af[8], bf[4];
                if (AMM) {
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        af[t] = *reinterpret_cast<const double*>(sa + (t >> 1) * 2048 +
                                                                 moff[t & 1][s]);
                } else {
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        af[t] = *reinterpret_cast<const double*>(sa + t * 1024 + koff[s]);
                }
#pragma unroll
                for (int n = 0; n < 4; ++n)
                    bf[n] = *reinterpret_cast<const double*>(sb + n * 1024 + koff[s]);
#pragma unroll
                for (int t = 0; t < 8; ++t)
#pragma unroll
                    for (int n = 0; n < 4; ++n) dmma(acc[t][n][0], acc[t][n][1], af[t], bf[n]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }

        // ---------------- epilogue ----------------
        const int tid = threadIdx.x;
        if (p.splits > 1) {
            double* dst = p.partial + static_cast<size_t>(u) * TILE_ELEMS;
#pragma unroll
            for (int t = 0; t < 8; ++t)
#pragma unroll
                for (int n = 0; n < 4; ++n)
#pragma unroll
                    for (int i = 0; i < 2; ++i)
                        dst[((t * 4 + n) * 2 + i) * (CWARPS * 32) + tid] = acc[t][n][i];
        } else if (kFastEpilogue && p.kind != KIND_SYRK && !p.beta_one && p.alpha == 1.0 && w.row0 + BM <= p.M &&
                   w.col0 + BN <= p.N) {
            // Interior tile, plain store (+ column scale, non-finite flag): the
            // per-element generic epilogue was ~5k SASS instructions per unit,
            // more than the main loop (ncu round 2: no-instruction stalls and
            // the NN kernel's 5% gap). Addresses: two per-lane column bases
            // (i = 0, 1) + compile-time row / column-group offsets.
            int r0l, c0l, r1l, c1l;
            slot_coord(AMM, 0, tid, r0l, c0l);  // (t, n, i) = (0, 0, 0)
            slot_coord(AMM, 1, tid, r1l, c1l);  // (0, 0, 1): same row, column of i = 1
            double* base0 = p.C + (w.row0 + r0l) + (w.col0 + c0l) * p.ldc;
            double* base1 = p.C + (w.row0 + r1l) + (w.col0 + c1l) * p.ldc;
            double sc[4][2];
#pragma unroll
            for (int n = 0; n < 4; ++n) {
                sc[n][0] = p.col_scale ? p.col_scale[w.col0 + c0l + 8 * n] : 1.0;
                sc[n][1] = p.col_scale ? p.col_scale[w.col0 + c1l + 8 * n] : 1.0;
            }
            bool bad = false;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                // row offset of accumulator row-group t relative to t = 0
                const int dr = AMM ? 16 * (t >> 1) + 4 * (t & 1) : 8 * t;
#pragma unroll
                for (int n = 0; n < 4; ++n) {
                    const int64_t off = dr + static_cast<int64_t>(8 * n) * p.ldc;
                    bad |= !isfinite(acc[t][n][0]) || !isfinite(acc[t][n][1]);
                    base0[off] = acc[t][n][0] * sc[n][0];
                    base1[off] = acc[t][n][1] * sc[n][1];
                }
            }
            if (bad && p.flag) atomicOr(p.flag, 1);
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t)
#pragma unroll
                for (int n = 0; n < 4; ++n)
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        int r, c;
                        slot_coord(AMM, (t * 4 + n) * 2 + i, tid, r, c);
                        store_out(p, w.row0 + r, w.col0 + c, acc[t][n][i]);
                    }
        }
    }
}

// Fixed-order split-K reduction: out = sum_{s=0}^{S-1} partial[s][tile].
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const Params p) {
    const int t = blockIdx.x;
    const int tid = threadIdx.x;
    Params q = p;
    if (p.utab) {  // work line: the tile's units are contiguous, summed in unit order
        const int u0 = static_cast<int>(p.tfirst[t]), u1 = static_cast<int>(p.tfirst[t + 1]);
        const Unit w = decode(q, u0);
        for (int idx = blockIdx.y * 8; idx < blockIdx.y * 8 + 8; ++idx) {
            double s = 0.0;
            for (int u = u0; u < u1; ++u) s += p.partial[static_cast<size_t>(u) * TILE_ELEMS + idx * 256 + tid];
            int r, c;
            if (w.diag)
                slot_coord_diag(idx, tid, r, c);
            else
                slot_coord(p.a_mmajor, idx, tid, r, c);
            store_out(p, w.row0 + r, w.col0 + c, s);
        }
        return;
    }
    // Recover the tile origin from any unit of this tile (split 0).
    const Unit w = decode(q, t);
    for (int idx = blockIdx.y * 8; idx < blockIdx.y * 8 + 8; ++idx) {
        double s = 0.0;
        const double* src = p.partial + static_cast<size_t>(t) * TILE_ELEMS + idx * 256 + tid;
        for (int sp = 0; sp < p.splits; ++sp)
            s += src[static_cast<size_t>(sp) * p.n_tiles * TILE_ELEMS];
        int r, c;
        slot_coord(p.a_mmajor, idx, tid, r, c);
        store_out(p, w.row0 + r, w.col0 + c, s);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        SVDK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
        if (!ptr || q != cudaDriverEntryPointSuccess)
            fail(SVDK_E_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// 2-D FP64 map over a column-major matrix: dim0 = rows (contiguous), dim1 = cols.
CUtensorMap make_map(const double* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box0,
                     uint32_t box1) {
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    cuuint32_t box[2] = {box0, box1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base),
                             dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SVDK_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

// 3-D view of an M-major operand with rows % 16 == 0: dims (16, cols, rows/16),
// box (16, BK, BM/16), so one TMA fills a whole BM x BK stage.
CUtensorMap make_map_mmajor3(const double* base, int64_t rows, int64_t cols, int64_t ld) {
    CUtensorMap m;
    cuuint64_t dims[3] = {16, static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows / 16)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 8, 128};
    cuuint32_t box[3] = {16, BK, BM / 16};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base),
                             dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(SVDK_E_CUDA, "cuTensorMapEncodeTiled (3d) failed: " + std::to_string(r));
    return m;
}

// Pick the k-split count S so (tiles x S) fills whole waves of the SMs.
int choose_splits(int n_tiles, int64_t K, int sms) {
    const int64_t k_steps = ceil_div(K, BK);
    const int max_s = static_cast<int>(std::min<int64_t>(std::max<int64_t>(1, k_steps / 8), 256));
    double best_eff = 0;
    int best = 1;
    for (int s = 1; s <= max_s; ++s) {
        const int64_t units = static_cast<int64_t>(n_tiles) * s;
        const double eff = static_cast<double>(units) / (ceil_div(units, sms) * sms);
        if (eff > best_eff + 0.02) {
            best_eff = eff;
            best = s;
        }
        if (best_eff > 0.97) break;
    }
    return best;
}

// Work line of a tall SYRK (see syrk): [units, (tile, k0, k1) x units, first unit
// of CTA 0..ctas, first unit of tile 0..n_tiles]. Tiles in the kernel's upper
// column-by-column order; a k-step of a diagonal tile weighs 17, of any other 32.
constexpr int64_t kSyrkLineMinRows = 32768;
// Weight of a diagonal tile's k-step against 32 for a full tile. The DMMA count says 17; measured on
// B200 (2^20 x 1024 Gram: 17 -> 33.8 ms, 18 -> 31.2, 19 -> 31.4, 20 -> 31.6, 23 -> 32.4, 32 -> 34.5; uniform
// split-K grid 35.4 ms) a diagonal k-step costs ~0.59 of a full one (18 operand loads for 17 DMMAs).
constexpr int kSyrkDiagWeight = 19;
std::vector<long long> build_syrk_line(int tiles, int64_t K, int ctas, int diag_weight) {
    const int n_tiles = tiles * (tiles + 1) / 2;
    const long long ks = ceil_div(K, BK);
    std::vector<int> weight(static_cast<size_t>(n_tiles), 32);
    for (int tj = 0; tj < tiles; ++tj) weight[static_cast<size_t>(tj * (tj + 1) / 2 + tj)] = diag_weight;
    long long total = 0;
    for (int w : weight) total += ks * w;
    // boundary b of the line, as (tile, k-step): the tile holding weight position b * total / ctas
    std::vector<long long> out;
    std::vector<long long> utab, cfirst(static_cast<size_t>(ctas) + 1), tfirst(static_cast<size_t>(n_tiles) + 1, -1);
    int tile = 0;
    long long step = 0, before = 0;  // weight before `tile`
    for (int b = 0; b < ctas; ++b) {
        cfirst[static_cast<size_t>(b)] = static_cast<long long>(utab.size() / 3);
        const long long hi = b + 1 == ctas ? total : static_cast<long long>((static_cast<__int128>(total) * (b + 1)) / ctas);
        while (tile < n_tiles) {
            const long long wt = weight[static_cast<size_t>(tile)];
            const long long tile_end = before + ks * wt;
            // last k-step of this tile that belongs to CTA b (rounded to a whole step)
            long long stop = hi >= tile_end ? ks : (hi - before + wt / 2) / wt;
            stop = std::max(stop, step);
            if (stop > step) {
                if (tfirst[static_cast<size_t>(tile)] < 0) tfirst[static_cast<size_t>(tile)] = static_cast<long long>(utab.size() / 3);
                utab.push_back(tile);
                utab.push_back(std::min<long long>(step * BK, K));
                utab.push_back(std::min<long long>(stop * BK, K));
                step = stop;
            }
            if (step < ks) break;  // the rest of this tile goes to the next CTA
            before = tile_end;
            ++tile;
            step = 0;
            if (hi <= before) break;
        }
    }
    cfirst[static_cast<size_t>(ctas)] = static_cast<long long>(utab.size() / 3);
    tfirst[static_cast<size_t>(n_tiles)] = static_cast<long long>(utab.size() / 3);
    for (int t = n_tiles - 1; t >= 0; --t)
        if (tfirst[static_cast<size_t>(t)] < 0) tfirst[static_cast<size_t>(t)] = tfirst[static_cast<size_t>(t) + 1];
    out.push_back(static_cast<long long>(utab.size() / 3));
    out.insert(out.end(), utab.begin(), utab.end());
    out.insert(out.end(), cfirst.begin(), cfirst.end());
    out.insert(out.end(), tfirst.begin(), tfirst.end());
    for (long long u = 0; u < out[0]; ++u) out.push_back(u);  // clist: every CTA's units are consecutive
    return out;
}

// The same table format for the lockstep variant: the uniform tiles x S k-chunks grid (one unit per CTA, all
// CTAs of a chunk walking the same k window, so a column block of A is fetched once for the tiles that share
// it), rebalanced by handing the last fraction g of every full unit's chunk, cut into sub-tails, to the CTAs of
// the cheaper diagonal units and to the CTAs the grid leaves without a unit (c4: 144 units on 148 SMs). Empty when the shape does not fit (fewer
// than two chunks per tile in one wave, or no off-diagonal tile).
std::vector<long long> build_syrk_lockstep(int tiles, int64_t K, int ctas, int diag_weight) {
    const int n_tiles = tiles * (tiles + 1) / 2, n_full = tiles * (tiles - 1) / 2, n_diag = tiles;
    const int S = ctas / n_tiles;
    const long long ks = ceil_div(K, BK);
    if (tiles < 2 || S < 2 || ks < 64LL * S) return {};
    // Helpers of the tails: the S n_diag diagonal CTAs (spare 1 - w_d / 32 of a unit each) and the
    // ctas - S n_tiles CTAs without a unit of their own. Balanced finish at T = 1 - g of a unit:
    //   n_full g = n_diag (T - w_d / 32) + F T,  F = free CTAs per chunk.
    const int n_free = ctas - S * n_tiles;
    const double wd = diag_weight / 32.0, F = static_cast<double>(n_free) / S;
    const double g = (n_diag * (1.0 - wd) + F) / (n_full + n_diag + F);
    constexpr int H = 16;  // sub-tails per full unit (a helper ends within half a sub-tail of the mean: ~0.4%)
    std::vector<char> is_diag(static_cast<size_t>(n_tiles), 0);
    for (int tj = 0; tj < tiles; ++tj) is_diag[static_cast<size_t>(tj * (tj + 1) / 2 + tj)] = 1;
    std::vector<long long> utab, tfirst(static_cast<size_t>(n_tiles) + 1);
    std::vector<long long> base_unit(static_cast<size_t>(n_tiles) * S);
    std::vector<std::pair<long long, long long>> tails;  // (k-steps, unit id)
    for (int t = 0; t < n_tiles; ++t) {
        tfirst[static_cast<size_t>(t)] = static_cast<long long>(utab.size() / 3);
        for (int sc = 0; sc < S; ++sc) {
            const long long c0 = ks * sc / S, c1 = ks * (sc + 1) / S;
            const long long tail = is_diag[static_cast<size_t>(t)] ? 0 : static_cast<long long>(g * (c1 - c0) + 0.5);
            auto push = [&](long long a, long long b) {
                utab.push_back(t);
                utab.push_back(std::min<long long>(a * BK, K));
                utab.push_back(std::min<long long>(b * BK, K));
                return static_cast<long long>(utab.size() / 3 - 1);
            };
            base_unit[static_cast<size_t>(t) * S + sc] = push(c0, c1 - tail);
            for (int i = 0; i < H && tail > 0; ++i) {
                const long long a = c1 - tail + tail * i / H, b = c1 - tail + tail * (i + 1) / H;
                if (b > a) tails.emplace_back(b - a, push(a, b));
            }
        }
    }
    tfirst[static_cast<size_t>(n_tiles)] = static_cast<long long>(utab.size() / 3);
    // CTA (chunk sc, tile t) = sc * n_tiles + t, then the free CTAs. Every sub-tail goes to the helper
    // with the least work so far (work in full-tile k-steps; longest sub-tails first).
    std::vector<std::vector<long long>> lists(static_cast<size_t>(ctas));
    std::vector<double> work(static_cast<size_t>(ctas), 0.0);
    std::vector<int> helpers;
    for (int sc = 0; sc < S; ++sc)
        for (int t = 0; t < n_tiles; ++t) {
            const int b = sc * n_tiles + t;
            const long long len = ks * (sc + 1) / S - ks * sc / S;
            lists[static_cast<size_t>(b)].push_back(base_unit[static_cast<size_t>(t) * S + sc]);
            if (is_diag[static_cast<size_t>(t)]) {
                work[static_cast<size_t>(b)] = wd * static_cast<double>(len);
                helpers.push_back(b);
            }
        }
    for (int b = S * n_tiles; b < ctas; ++b) helpers.push_back(b);
    std::stable_sort(tails.begin(), tails.end(),
                     [](const std::pair<long long, long long>& x, const std::pair<long long, long long>& y) {
                         return x.first > y.first;
                     });
    for (const auto& tl : tails) {
        int best = helpers[0];
        for (int hb : helpers)
            if (work[static_cast<size_t>(hb)] < work[static_cast<size_t>(best)]) best = hb;
        lists[static_cast<size_t>(best)].push_back(tl.second);
        work[static_cast<size_t>(best)] += static_cast<double>(tl.first);
    }
    std::vector<long long> out, cfirst(static_cast<size_t>(ctas) + 1), clist;
    for (int b = 0; b < ctas; ++b) {
        cfirst[static_cast<size_t>(b)] = static_cast<long long>(clist.size());
        clist.insert(clist.end(), lists[static_cast<size_t>(b)].begin(), lists[static_cast<size_t>(b)].end());
    }
    cfirst[static_cast<size_t>(ctas)] = static_cast<long long>(clist.size());
    out.push_back(static_cast<long long>(utab.size() / 3));
    out.insert(out.end(), utab.begin(), utab.end());
    out.insert(out.end(), cfirst.begin(), cfirst.end());
    out.insert(out.end(), tfirst.begin(), tfirst.end());
    out.insert(out.end(), clist.begin(), clist.end());
    return out;
}

bool tma_ok(const void* p, int64_t ld) {
    return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 2 == 0);
}

void launch(Ctx* c, Params& p, const CUtensorMap& ma, const CUtensorMap& mb) {
    ensure_smem_attr(reinterpret_cast<const void*>(gemm_kernel<false>), SMEM_BYTES);
    ensure_smem_attr(reinterpret_cast<const void*>(gemm_kernel<true>), SMEM_BYTES);
    ensure_smem_attr(reinterpret_cast<const void*>(gemm_kernel<false, true>), SMEM_BYTES);
    DBuf partial;
    if (p.splits > 1) {
        partial = DBuf(c, static_cast<size_t>(p.units) * TILE_ELEMS);
        p.partial = partial.p();
    }
    const int grid = p.utab ? c->num_sms : std::min(p.units, c->num_sms);
    // algorithmic work: Gram m n (n+1); GEMM 2 M N K
    const double flops = p.kind == KIND_SYRK ? static_cast<double>(p.K) * p.M * (p.M + 1)
                         : p.b_upper      ? 1.0 * p.M * p.N * (p.N + 1)  // triangular B: M N (N+1)
                                          : 2.0 * p.M * p.N * p.K;
    const double bytes = p.kind == KIND_SYRK ? 8.0 * (p.K * p.M + p.M * p.M)
                                             : 8.0 * (p.M * p.K + p.K * p.N + p.M * p.N);
    {
        // one phase per kernel form, so bench.py can report the dominant one
        PhaseTimer timer(c, p.kind == KIND_SYRK ? "dmma_syrk" : (p.a_mmajor ? "dmma_gemm_nn" : "dmma_gemm_tn"),
                         flops, bytes);
        if (p.a_mmajor)
            gemm_kernel<true><<<grid, THREADS, SMEM_BYTES, c->stream>>>(ma, mb, p);
        else if (p.utab)
            gemm_kernel<false, true><<<grid, THREADS, SMEM_BYTES, c->stream>>>(ma, mb, p);
        else
            gemm_kernel<false><<<grid, THREADS, SMEM_BYTES, c->stream>>>(ma, mb, p);
        SVDK_CHECK_LAUNCH();
        c->launches++;
    }
    if (p.splits > 1) {
        PhaseTimer timer(c, "splitk_reduce", 0.0, 8.0 * p.units * TILE_ELEMS);
        splitk_reduce_kernel<<<dim3(p.n_tiles, 8), 256, 0, c->stream>>>(p);
        SVDK_CHECK_LAUNCH();
        c->launches++;
    }
}

// ---------------------------------------------------------------------------
// Compact small-K GEMM / SYRK (K <= 128): the Cholesky / triangular-inverse
// panel updates (K = 64) are a few tiles each, and a one-tile launch of the
// big TMA/mbarrier kernel above costs ~40 us, mostly instruction fetch for its
// fully unrolled body (ncu: `no_instruction` stalls). This kernel is small:
// 64 x 64 output tiles, 4 warps of 32 x 32 (m8n8k4 DMMA), operands staged in
// shared memory 16 k at a time with plain coalesced loads. Same epilogue
// semantics as store_out (flag, column scale, alpha, beta, SYRK mirror).
// ---------------------------------------------------------------------------
constexpr int ST = 64, SK = 16, SLD = ST + 4;

__global__ void __launch_bounds__(128)
    gemm_small_kernel(int kind, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                      int64_t ldb, double* C, int64_t ldc, double alpha, int beta_one, const double* col_scale,
                      int* flag, int tiles_n) {
    __shared__ double As[SK][SLD], Bs[SK][SLD];
    const int ti = blockIdx.x / tiles_n, tj = blockIdx.x % tiles_n;
    if (kind == KIND_SYRK && ti > tj) return;  // upper tiles only; mirrored in the epilogue
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, r = lane >> 2, kq = lane & 3;
    const int wm = w & 1, wn = w >> 1;
    const int64_t row0 = static_cast<int64_t>(ti) * ST, col0 = static_cast<int64_t>(tj) * ST;
    const double* Bm = kind == KIND_SYRK ? A : B;
    const int64_t ldbm = kind == KIND_SYRK ? lda : ldb;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int64_t k0 = 0; k0 < K; k0 += SK) {
        // A chunk -> As[k][m]: NN reads A[m + k lda] (m fastest), TN / SYRK A[k + m lda] (k fastest)
#pragma unroll
        for (int it = 0; it < SK * ST / 128; ++it) {
            const int e = tid + it * 128;
            int kk, mm;
            if (kind == KIND_NN) {
                mm = e % ST;
                kk = e / ST;
            } else {
                kk = e % SK;
                mm = e / SK;
            }
            const int64_t gm = row0 + mm, gk = k0 + kk;
            double v = 0.0;
            if (gm < M && gk < K) v = kind == KIND_NN ? A[gm + gk * lda] : A[gk + gm * lda];
            As[kk][mm] = v;
            const int64_t gn = col0 + e / SK;
            const int kb = e % SK;
            double u = 0.0;
            if (gn < N && k0 + kb < K) u = Bm[(k0 + kb) + gn * ldbm];
            Bs[kb][e / SK] = u;
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < SK / 4; ++ks) {
            double af[4], bf[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) af[a] = As[4 * ks + kq][32 * wm + 8 * a + r];
#pragma unroll
            for (int b = 0; b < 4; ++b) bf[b] = Bs[4 * ks + kq][32 * wn + 8 * b + r];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int64_t row = row0 + 32 * wm + 8 * a + r, col = col0 + 32 * wn + 8 * b + 2 * kq + i;
                if (row >= M || col >= N) continue;
                double v = acc[a][b][i];
                if (kind == KIND_SYRK) {
                    if (row > col) continue;  // one value per mirror pair -> exact symmetry
                    if (alpha != 1.0) v *= alpha;
                    if (beta_one) v += C[row + col * ldc];
                    C[row + col * ldc] = v;
                    C[col + row * ldc] = v;
                    continue;
                }
                if (flag && !isfinite(v)) atomicOr(flag, 1);
                if (col_scale) v *= col_scale[col];
                if (alpha != 1.0) v *= alpha;
                if (beta_one) v += C[row + col * ldc];
                C[row + col * ldc] = v;
            }
}

// Small-K problems go to gemm_small_kernel (measured: see DESIGN 3.3).
bool small_k(int64_t m, int64_t n, int64_t k) {
    static const bool on = [] {
        const char* e = std::getenv("SVDK_SMALL_GEMM");
        return !(e && e[0] == '0');
    }();
    return on && k <= 128 && m * n <= (int64_t{1} << 22);
}

void launch_small(Ctx* c, int kind, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                  const double* B, int64_t ldb, double* C, int64_t ldc, double alpha, bool beta_one,
                  const double* col_scale, int* flag) {
    const int tiles_m = static_cast<int>(ceil_div(M, ST)), tiles_n = static_cast<int>(ceil_div(N, ST));
    const double flops = kind == KIND_SYRK ? static_cast<double>(K) * M * (M + 1) : 2.0 * M * N * K;
    const double bytes = kind == KIND_SYRK ? 8.0 * (K * M + M * M) : 8.0 * (M * K + K * N + M * N);
    PhaseTimer timer(c, "dmma_gemm_small", flops, bytes);
    gemm_small_kernel<<<tiles_m * tiles_n, 128, 0, c->stream>>>(kind, M, N, K, A, lda, B, ldb, C, ldc, alpha,
                                                                beta_one ? 1 : 0, col_scale, flag, tiles_n);
    SVDK_CHECK_LAUNCH();
    c->launches++;
}

}  // namespace

CUtensorMap tensor_map_2d(const double* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box0,
                          uint32_t box1, CUtensorMapSwizzle swizzle) {
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    cuuint32_t box[2] = {box0, box1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SVDK_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

void syrk(Ctx* c, int64_t m, int64_t n, const double* A, int64_t lda, double* G, int64_t ldg,
          double alpha, bool beta_one) {
    if (n == 0) return;
    if (m == 0) {
        if (!beta_one)
            for (int64_t j = 0; j < n; ++j) fill(c, G + j * ldg, n, 0.0);
        return;
    }
    if (small_k(n, n, m)) {
        launch_small(c, KIND_SYRK, n, n, m, A, lda, nullptr, 0, G, ldg, alpha, beta_one, nullptr, nullptr);
        return;
    }
    DBuf padded;
    if (!tma_ok(A, lda)) {
        const int64_t ld2 = round_up(m, 2);
        padded = DBuf(c, static_cast<size_t>(ld2) * n);
        copy_mat(c, A, lda, padded.p(), ld2, m, n);
        A = padded.p();
        lda = ld2;
    }
    Params p{};
    p.kind = KIND_SYRK;
    p.a_mmajor = 0;
    p.M = n;
    p.N = n;
    p.K = m;
    p.tiles_m = p.tiles_n = static_cast<int>(ceil_div(n, BM));
    p.n_tiles = p.tiles_m * (p.tiles_m + 1) / 2;
    int s = choose_splits(p.n_tiles, m, c->num_sms);
    p.k_per_split = round_up(ceil_div(m, s), BK);
    p.splits = static_cast<int>(ceil_div(m, p.k_per_split));
    p.units = p.n_tiles * p.splits;
    p.C = G;
    p.ldc = ldg;
    p.alpha = alpha;
    p.beta_one = beta_one ? 1 : 0;
    // Tall Gram (m >= kSyrkLineMinRows): a table of (tile, k0, k1) units instead of the uniform tiles x
    // splits grid, in which a diagonal tile computes only its 136 upper 8 x 8 blocks (17 / 32 of a tile's
    // DMMAs; diag_unit) and its k-steps weigh kSyrkDiagWeight against 32:
    //   default   the lockstep table where the shape fits it (>= 2 k-chunks per tile in one wave: n <= ~1400;
    //             c2 / c4): the uniform k-chunk grid — all CTAs of a chunk walk the same k window, so a
    //             column block of A is fetched once for the tiles sharing it — with the last 9% of every
    //             full unit's chunk handed to the CTAs of the cheaper diagonal units; else the uniform grid
    //   =1        the work line: all k-steps of all tiles end to end, cut into equal-weight contiguous
    //             pieces per CTA (pieces may straddle two tiles). 3-5% faster than the default on the Gram,
    //             but the pieces sit at unrelated k offsets and A is re-fetched per tile: 7x (n = 1024) to
    //             30x (n = 4096) the algorithmic DRAM reads
    //   =0        always the uniform grid
    // The per-unit partial tiles are summed per tile in unit order (fixed order, exact mirror).
    DBuf line;
    const char* sk_env = std::getenv("SVDK_SYRK_LINE");
    const int sk_mode = sk_env ? std::atoi(sk_env) : 2;
    if (m >= kSyrkLineMinRows && sk_mode != 0) {
        const char* dw_env = std::getenv("SVDK_SYRK_DIAGW");
        const int diag_w = dw_env ? std::min(32, std::max(1, std::atoi(dw_env))) : kSyrkDiagWeight;
        std::vector<long long> host = sk_mode == 1 ? build_syrk_line(p.tiles_m, m, c->num_sms, diag_w)
                                                   : build_syrk_lockstep(p.tiles_m, m, c->num_sms, diag_w);
        if (!host.empty()) {
            const size_t units = static_cast<size_t>(host[0]);
            line = DBuf(c, host.size());
            h2d(c, line.p(), reinterpret_cast<const double*>(host.data()), static_cast<int64_t>(host.size()));
            const long long* base = reinterpret_cast<const long long*>(line.p());
            p.utab = base + 1;
            p.cfirst = p.utab + 3 * units;
            p.tfirst = p.cfirst + c->num_sms + 1;
            p.clist = p.tfirst + p.n_tiles + 1;
            p.units = static_cast<int>(units);
            p.splits = 2;  // partial tiles + the reduction kernel
        }
    }
    const CUtensorMap ma = make_map(A, m, n, lda, BK, BM);
    launch(c, p, ma, ma);
}

void gemm(Ctx* c, bool transa, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
          const double* B, int64_t ldb, double* C, int64_t ldc, const double* col_scale,
          bool nonfinite_check, double alpha, bool beta_one, bool b_upper) {
    if (m == 0 || n == 0) return;
    if (k == 0) {
        if (!beta_one)
            for (int64_t j = 0; j < n; ++j) fill(c, C + j * ldc, m, 0.0);
        return;
    }
    if (!b_upper && small_k(m, n, k)) {
        launch_small(c, transa ? KIND_TN : KIND_NN, m, n, k, A, lda, B, ldb, C, ldc, alpha, beta_one, col_scale,
                     nonfinite_check ? c->d_flags : nullptr);
        return;
    }
    DBuf pa, pb;
    if (!tma_ok(A, lda)) {
        const int64_t rows = transa ? k : m, cols = transa ? m : k;
        const int64_t ld2 = round_up(rows, 2);
        pa = DBuf(c, static_cast<size_t>(ld2) * cols);
        copy_mat(c, A, lda, pa.p(), ld2, rows, cols);
        A = pa.p();
        lda = ld2;
    }
    if (!tma_ok(B, ldb)) {
        const int64_t ld2 = round_up(k, 2);
        pb = DBuf(c, static_cast<size_t>(ld2) * n);
        copy_mat(c, B, ldb, pb.p(), ld2, k, n);
        B = pb.p();
        ldb = ld2;
    }
    Params p{};
    p.kind = transa ? KIND_TN : KIND_NN;
    p.a_mmajor = transa ? 0 : 1;
    p.M = m;
    p.N = n;
    p.K = k;
    p.tiles_m = static_cast<int>(ceil_div(m, BM));
    p.tiles_n = static_cast<int>(ceil_div(n, BN));
    p.n_tiles = p.tiles_m * p.tiles_n;
    int s = 1;
    if (p.n_tiles < 2 * c->num_sms) s = choose_splits(p.n_tiles, k, c->num_sms);
    p.k_per_split = round_up(ceil_div(k, s), BK);
    p.splits = static_cast<int>(ceil_div(k, p.k_per_split));
    p.units = p.n_tiles * p.splits;
    p.C = C;
    p.ldc = ldc;
    p.col_scale = col_scale;
    p.alpha = alpha;
    p.beta_one = beta_one ? 1 : 0;
    p.b_upper = b_upper ? 1 : 0;
    if (nonfinite_check) p.flag = c->d_flags;  // sticky; see raise_if_nonfinite()
    static const bool tma3 = [] {
        const char* e = std::getenv("SVDK_NN_TMA3");
        return !(e && e[0] == '0');
    }();
    p.a_tma3 = (!transa && tma3 && m % 16 == 0) ? 1 : 0;
    const CUtensorMap ma = transa     ? make_map(A, k, m, lda, BK, BM)
                           : p.a_tma3 ? make_map_mmajor3(A, m, k, lda)
                                      : make_map(A, m, k, lda, 16, BK);
    const CUtensorMap mb = make_map(B, k, n, ldb, BK, BN);
    launch(c, p, ma, mb);
}

}  // namespace svdk

// Development / test hook (not part of the public ABI): the SYRK work line
// for `tiles` x `tiles` upper tiles, K rows and `ctas` CTAs. Returns the
// table's length in 64-bit words; copies it when it fits `cap`.
extern "C" long long svdk_debug_syrk_line(int tiles, long long K, int ctas, int diag_weight, long long* out,
                                          long long cap) {
    if (tiles < 1 || K < 1 || ctas < 1) return -1;
    // diag_weight < 0: the lockstep variant with weight -diag_weight (0 entries when the shape does not fit)
    const std::vector<long long> t =
        diag_weight < 0 ? svdk::build_syrk_lockstep(tiles, K, ctas, -diag_weight)
                        : svdk::build_syrk_line(tiles, K, ctas, diag_weight > 0 ? diag_weight : svdk::kSyrkDiagWeight);
    if (out && static_cast<long long>(t.size()) <= cap) std::copy(t.begin(), t.end(), out);
    return static_cast<long long>(t.size());
}
