// jacobi.cu — parallel block-cyclic Jacobi eigensolver for symmetric n x n.
//
// Replaces eig_sym (reference kernels.cpp:241-346) and keeps its contract:
//   * square input, else DimensionError                        (:247-249)
//   * max|s - s^T| <= 1e-8 max|s|, else ParamError              (:251-262)
//   * iterate on (s + s^T)/2                                     (:264-269)
//   * converged when off(A) = sqrt(2 sum_{i>j} a_ij^2) <= 1e-12 ||A||_F,
//     tested before the first sweep and after every sweep         (:271-274, :319)
//   * rotation formulas tau, t, c, s of the reference             (:282-290)
//   * sweep cap (default 30) -> NumericalError(off(A))            (:321-326)
//   * eigenvalues = final diagonal, STABLE descending sort        (:328-331)
//
// Parallel ordering instead of cyclic-by-row: the n indices are cut into nb
// blocks of b; a sweep is nb-1 rounds of a round-robin tournament over the
// blocks, and in each round the nb/2 disjoint block pairs (I, J) are
// processed at once:
//   1. jacobi_pair_solve: one CTA per pair diagonalises the 2b x 2b
//      subproblem A[IJ, IJ] in shared memory with the reference rotations
//      (itself in parallel round-robin order, b rotations at a time), and
//      emits the accumulated rotation Q_p (2b x 2b).
//   2. jacobi_update: every off-diagonal pair block becomes
//      A[IJ_p, IJ_q] <- Q_p^T A[IJ_p, IJ_q] Q_q (written with its mirror, so A
//      stays exactly symmetric) and V[:, IJ_q] <- V[:, IJ_q] Q_q, as small
//      FP64 DMMA GEMMs out of shared memory.
// A sweep therefore applies every rotation of a cyclic sweep's pair set, in
// block form, with ~8 n^3 flops on the DMMA pipe. Padding indices (n rounded
// up to a multiple of 2b) carry zero rows/columns, never couple, and are
// dropped at the end.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "svdk_internal.h"

namespace svdk {
namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Round-robin (circle method) pairing of P players, round r, pair i.
__host__ __device__ __forceinline__ void circle_pair(int P, int r, int i, int& a, int& b) {
    const int m = P - 1;
    a = (i == 0) ? 0 : ((i - 1 + r) % m) + 1;
    b = ((P - 2 - i + r) % m) + 1;
    if (a > b) {
        const int t = a;
        a = b;
        b = t;
    }
}

// Jacobi rotation annihilating a_pq (reference kernels.cpp:282-290):
//   tau = (a_qq - a_pp) / (2 a_pq), t = sgn(tau) / (|tau| + sqrt(1 + tau^2)),
//   c = 1 / sqrt(1 + t^2), s = t c.
// Evaluated in the algebraically identical division-free form
//   d = a_qq - a_pp, e = 2 a_pq, D = |d| + sqrt(d^2 + e^2),
//   c = D / sqrt(D^2 + e^2), s = sgn(tau) |e| / sqrt(D^2 + e^2)
// with two FP64 reciprocal square roots: 209 cycles of dependent latency on
// B200 vs 544 for the reference's 2 sqrt + 3 div (tools/probes/rot_latency.cu),
// and this chain is the serial part of every inner round. eig_sym prescales
// the matrix by a power of two so d^2 + e^2 cannot overflow or underflow.
// The accumulated Q is re-orthogonalised after the inner sweep, so last-ulp
// differences in c, s do not accumulate.
__device__ __forceinline__ void rotation(double app, double aqq, double apq, double& c, double& s) {
    const double d = aqq - app, e = 2.0 * apq;
    const double r2 = fma(d, d, e * e);
    const double D = fabs(d) + r2 * rsqrt(r2);  // |d| + sqrt(d^2 + e^2)
    const double inv = rsqrt(fma(D, D, e * e));
    c = D * inv;
    s = (d > 0.0 ? e : (d < 0.0 ? -e : fabs(e))) * inv;  // tau = +-0 -> t = +1
}

// Global index of local index i (0..2b-1) of the pair (I, J).
__device__ __forceinline__ int64_t gidx(int B, int I, int J, int i) {
    return i < B ? static_cast<int64_t>(I) * B + i : static_cast<int64_t>(J) * B + (i - B);
}

// C = op(A) * B on TB x TB shared-memory matrices (col-major, ld TB+4) with
// FP64 DMMA; result is written to C (same layout). No block barrier inside.
// smem_mma_t: the same, run by the `nthr` threads tid in [0, nthr) of a
// thread group (warp-aligned) instead of the whole block.
template <int TB, bool TRANS_A>
__device__ __forceinline__ void smem_mma_t(const double* A, const double* Bm, double* C, int tid, int nthr) {
    constexpr int LD = TB + 4;
    constexpr int NT = TB / 8;
    constexpr int WTM = NT >= 8 ? 2 : 1;
    constexpr int WTN = NT >= 8 ? 4 : (NT >= 4 ? 2 : 1);
    constexpr int WARPS_M = NT / WTM, WARPS_N = NT / WTN;
    static_assert(WARPS_M * WARPS_N <= 8, "tile split");
    const int lane = tid & 31, nwarps = nthr >> 5;
    const int r = lane >> 2, kq = lane & 3;
    for (int wt = tid >> 5; wt < WARPS_M * WARPS_N; wt += nwarps) {
        const int wm = wt % WARPS_M, wn = wt / WARPS_M;
        double acc[WTM][WTN][2];
#pragma unroll
        for (int a = 0; a < WTM; ++a)
#pragma unroll
            for (int b = 0; b < WTN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
        for (int k0 = 0; k0 < TB; k0 += 4) {
            const int k = k0 + kq;
            double af[WTM], bf[WTN];
#pragma unroll
            for (int a = 0; a < WTM; ++a) {
                const int m = (wm * WTM + a) * 8 + r;
                af[a] = TRANS_A ? A[k + m * LD] : A[m + k * LD];
            }
#pragma unroll
            for (int b = 0; b < WTN; ++b) {
                const int nn = (wn * WTN + b) * 8 + r;
                bf[b] = Bm[k + nn * LD];
            }
#pragma unroll
            for (int a = 0; a < WTM; ++a)
#pragma unroll
                for (int b = 0; b < WTN; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
#pragma unroll
        for (int a = 0; a < WTM; ++a)
#pragma unroll
            for (int b = 0; b < WTN; ++b) {
                const int row = (wm * WTM + a) * 8 + r;
                const int col = (wn * WTN + b) * 8 + 2 * kq;
                C[row + col * LD] = acc[a][b][0];
                C[row + (col + 1) * LD] = acc[a][b][1];
            }
    }
}

template <int TB, bool TRANS_A>
__device__ __forceinline__ void smem_mma(const double* A, const double* Bm, double* C) {
    smem_mma_t<TB, TRANS_A>(A, Bm, C, threadIdx.x, blockDim.x);
}

// ---------------------------------------------------------------------------
// 1. per-pair subproblem solve
// ---------------------------------------------------------------------------
// One CTA diagonalises M = A[IJ, IJ] (TB x TB) in shared memory and emits the
// accumulated rotation Q. Each inner round applies TB/2 disjoint rotations
// (round-robin pairs) as ONE fused phase: every 2x2 block (rows {p_i,q_i}) x
// (cols {p_j,q_j}) is replaced by R_i^T B R_j, so a round costs one barrier
// after the rotation parameters and one after the update. Inner sweeps stop
// when no |m_pq| exceeds skip_tau. A pair whose subproblem is already
// diagonal to skip_tau is flagged inactive (Q = I) and its blocks skipped.
// M itself is scratch: the update kernel applies the (re-orthogonalised) Q to
// every pair block, the diagonal ones included, so A changes by one
// similarity per round.
// Development probe: clock64 stamps of CTA 0 in the last pair solve (read by
// svdk_debug_jacobi_probe; not part of the public ABI).
__device__ long long g_jprobe[16];
// %globaltimer stamps of the fused round kernels' roles per round (SVDK_PROBES builds, tools/fr_timeline.py)
__device__ unsigned long long g_jtimeline[16 * 8];
#ifdef SVDK_PROBES
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

template <int TB>
constexpr int solve_q_warps() {
    // Q <- Q J is split over warps by rows (TB = 32: 4 warps x 8 rows): one warp
    // doing all 32 rows was a ~1k-cycle shuffle/FP64 chain per inner round
    return TB == 32 ? 4 : 1;
}
template <int TB>
constexpr int solve_threads() {
    // M threads (one 2x2 block each) + the Q warps (Q in registers) + 1 lookahead warp
    return (TB / 2) * (TB / 2) + 32 * solve_q_warps<TB>() + 32;
}

// R_i^T B R_j on the 2x2 block B = [[m00, m01], [m10, m11]] of rows (p_i, q_i)
// and columns (p_j, q_j); s == 0 marks an identity rotation; `same` (i == j)
// annihilates the rotated pair exactly. Written with explicit fma so every
// thread that evaluates the same block gets the same bits.
__device__ __forceinline__ void xform2x2(double& m00, double& m01, double& m10, double& m11,
                                         double ci, double si, double cj, double sj, bool same) {
    // Branch-free: a skipped rotation has (c, s) = (1, 0) and the fma forms
    // below then return their input (up to the sign of a zero), so lanes whose
    // rotations are skipped no longer diverge from the rest of the warp.
    {  // columns
        const double a0 = fma(cj, m00, -(sj * m01)), b0 = fma(sj, m00, cj * m01);
        const double a1 = fma(cj, m10, -(sj * m11)), b1 = fma(sj, m10, cj * m11);
        m00 = a0; m01 = b0; m10 = a1; m11 = b1;
    }
    {  // rows
        const double a0 = fma(ci, m00, -(si * m10)), b0 = fma(si, m00, ci * m10);
        const double a1 = fma(ci, m01, -(si * m11)), b1 = fma(si, m01, ci * m11);
        m00 = a0; m10 = b0; m01 = a1; m11 = b1;
    }
    const bool zero = same && si != 0.0;  // the rotated pair itself is annihilated
    m01 = zero ? 0.0 : m01;
    m10 = zero ? 0.0 : m10;
}

// Entry (u, v) of R_i^T B R_j alone, in xform2x2's operation order (columns
// first, then rows; branch-free like xform2x2, so the three entries of a
// lookahead are evaluated side by side and equal the M threads' values).
__device__ __forceinline__ double xform_entry_nb(double m00, double m01, double m10, double m11, double ci,
                                                 double si, double cj, double sj, int u, int v) {
    const double xc = v ? sj : cj, yc = v ? cj : -sj;
    const double t0 = fma(xc, m00, yc * m01), t1 = fma(xc, m10, yc * m11);
    const double xr = u ? si : ci, yr = u ? ci : -si;
    return fma(xr, t0, yr * t1);
}

// Programmatic dependent launch (PDL) inside a Jacobi round chain
// (solve -> A update -> next solve on one stream): the successor is launched
// with the programmatic-serialisation attribute, so its launch overlaps the
// predecessor's tail and it runs its independent prologue (the solve's
// schedule tables) before pdl_wait(), which returns once the predecessor grid
// has completed and its memory is visible (a no-op without the attribute).
// An explicit early trigger (griddepcontrol.launch_dependents at kernel
// start, -DSVDK_PDL_TRIGGER) measured mixed: eig(256) 3.20 -> 3.12 ms and
// eig(2048) 54.1 -> 50.4 ms, but eig(512) 6.2 -> 7.4 ms and eig(1024) 13.8 ->
// 16.4 ms (the early-resident waiting CTAs crowd the running grid), so the
// implicit trigger at grid completion is used. Without PDL: 3.28 / 6.31 /
// 15.6 / 54.0 ms for n = 256 / 512 / 1024 / 2048.
__device__ __forceinline__ void pdl_trigger() {
#ifdef SVDK_PDL_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// barrier over n threads that also ORs a predicate across them
__device__ __forceinline__ bool named_bar_or(int id, int n, bool pred) {
    unsigned out;
    asm volatile(
        "{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n bar.red.or.pred q, %2, %3, p;\n selp.u32 %0, 1, 0, q;\n}\n"
        : "=r"(out)
        : "r"(static_cast<unsigned>(pred)), "r"(id), "r"(n)
        : "memory");
    return out != 0;
}

// The lookahead warp's part of an inner round: look_load fetches what
// rotation `lane` of round rr+1 needs from M_rr and round rr's rotations;
// look_finish forms the three entries of M_rr+1 (branch-free, so the three
// are evaluated side by side) and the rotation. Measured per inner round
// (clock64, tools/exp_pair.sh + tools/exp_probe.py): 1470 -> 1260 cycles with
// the branch-free entries. Gating the M threads and Q warps on a named barrier
// behind the lookahead's reads cut those reads from ~1.5k to ~600 cycles but
// moved the contention into the rotation (round 1375 cycles), so it is not used.
struct LookRead {
    double a00, a01, a10, a11, b00, b01, b10, b11, x00, x01, x10, x11, cp, sp, cq, sq;
    int rp, rq;
};
template <int LD, class Tabs>
__device__ __forceinline__ LookRead look_load(const Tabs& st, const double* M, double (*cs)[Tabs::kNP],
                                              double (*sn)[Tabs::kNP], int rr, int lane,
                                              long long* probe_look = nullptr, long long t0 = 0) {
    LookRead r;
    const unsigned long long d = st.look[rr][lane];
#ifdef SVDK_PROBES
    if (probe_look) {
        unsigned long long u;
        asm volatile("add.u64 %0, %1, 1;" : "=l"(u) : "l"(d));
        probe_look[0] = SVDK_CLOCK() - t0;
        probe_look[1] = static_cast<long long>(u);
    }
#endif
    const int bp = d & 31, bq = (d >> 5) & 31;
    r.rp = (d >> 10) & 1;
    r.rq = (d >> 11) & 1;
    const int p1 = (d >> 12) & 31, q1 = (d >> 17) & 31;
    const int p2 = (d >> 22) & 31, q2 = (d >> 27) & 31;
    r.cp = cs[rr][bp];
    r.sp = sn[rr][bp];
    r.cq = cs[rr][bq];
    r.sq = sn[rr][bq];
    // diagonal blocks (bp, bp), (bq, bq) and the coupling block (bp, bq)
    r.a00 = M[p1 + p1 * LD]; r.a01 = M[p1 + q1 * LD]; r.a10 = M[q1 + p1 * LD]; r.a11 = M[q1 + q1 * LD];
    r.b00 = M[p2 + p2 * LD]; r.b01 = M[p2 + q2 * LD]; r.b10 = M[q2 + p2 * LD]; r.b11 = M[q2 + q2 * LD];
    r.x00 = M[p1 + p2 * LD]; r.x01 = M[p1 + q2 * LD]; r.x10 = M[q1 + p2 * LD]; r.x11 = M[q1 + q2 * LD];
    return r;
}
__device__ __forceinline__ void look_finish(const LookRead& r, double skip_tau, double& c, double& s) {
    // only the three entries the new rotation needs (branch-free form of
    // xform2x2's operation order, see xform_entry_nb)
    const double app = xform_entry_nb(r.a00, r.a01, r.a10, r.a11, r.cp, r.sp, r.cp, r.sp, r.rp, r.rp);
    const double aqq = xform_entry_nb(r.b00, r.b01, r.b10, r.b11, r.cq, r.sq, r.cq, r.sq, r.rq, r.rq);
    const double x = xform_entry_nb(r.x00, r.x01, r.x10, r.x11, r.cp, r.sp, r.cq, r.sq, r.rp, r.rq);
    c = 1.0;
    s = 0.0;
    if (fabs(x) > skip_tau) rotation(app, aqq, x, c, s);
}

// Inner schedule of a 2b subproblem for one mode (identical for every pair
// and round, so built once per eig_sym by jacobi_tables_kernel):
//   ptab[r][i]  rotation i of inner round r, packed p | q << 8
//   pinv[r][x]  pair holding index x in round r | role << 7 (role 1 = q)
//   look[r][i]  for rotation i of round r+1 = (p, q): the round-r pairs bp, bq
//               holding p and q, their roles and their (row, col) indices —
//               bits 0-4 bp, 5-9 bq, 10 role_p, 11 role_q, 12-16 p_bp,
//               17-21 q_bp, 22-26 p_bq, 27-31 q_bq (one LDS for the lookahead)
//   part[r][x]  the index paired with x in round r | role << 7
template <int TB>
struct __align__(16) SolveTables {
    static constexpr int kNP = TB / 2;
    unsigned long long look[TB - 1][TB / 2];
    int ptab[TB - 1][TB / 2];
    unsigned char pinv[TB - 1][TB];
    unsigned char part[TB - 1][TB];  // partner of index x in round r | role << 7 (one-sided solve)
};
static_assert(sizeof(SolveTables<32>) % 16 == 0 && sizeof(SolveTables<16>) % 16 == 0, "uint4 copy");

// modes 0 (all pairs), 1 (pairs inside each half), 2 (cross pairs): one CTA each
template <int TB>
__global__ void jacobi_tables_kernel(SolveTables<TB>* out) {
    constexpr int B = TB / 2, NP = TB / 2;
    const int mode = blockIdx.x;
    const int R = mode == 0 ? TB - 1 : (mode == 1 ? B - 1 : B);
    __shared__ SolveTables<TB> t;
    for (int e = threadIdx.x; e < (TB - 1) * NP; e += blockDim.x) {
        t.ptab[e / NP][e % NP] = 0;
        t.look[e / NP][e % NP] = 0;
    }
    for (int e = threadIdx.x; e < (TB - 1) * TB; e += blockDim.x) {
        t.pinv[e / TB][e % TB] = 0;
        t.part[e / TB][e % TB] = 0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * NP; e += blockDim.x) {
        int p, q;
        const int r = e / NP, i = e % NP;
        if (mode == 0) {
            circle_pair(TB, r, i, p, q);
        } else if (mode == 1) {  // round robin inside each half
            const int half = NP / 2, blk = i / half;
            circle_pair(B, r, i % half, p, q);
            p += blk * B;
            q += blk * B;
        } else {  // cross pairs: I_i with J_{(i + r) mod b}
            p = i;
            q = B + (i + r) % B;
        }
        t.ptab[r][i] = p | (q << 8);
        t.pinv[r][p] = static_cast<unsigned char>(i);
        t.pinv[r][q] = static_cast<unsigned char>(i | 128);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * NP; e += blockDim.x) {
        const int rr = e / NP, i = e % NP, nr = (rr + 1) % R;
        const int code = t.ptab[nr][i];
        const int ip = t.pinv[rr][code & 255], iq = t.pinv[rr][code >> 8];
        const int bp = ip & 127, bq = iq & 127;
        t.look[rr][i] =
            static_cast<unsigned long long>(bp) | (static_cast<unsigned long long>(bq) << 5) |
            (static_cast<unsigned long long>(ip >> 7) << 10) |
            (static_cast<unsigned long long>(iq >> 7) << 11) |
            (static_cast<unsigned long long>(t.ptab[rr][bp] & 255) << 12) |
            (static_cast<unsigned long long>(t.ptab[rr][bp] >> 8) << 17) |
            (static_cast<unsigned long long>(t.ptab[rr][bq] & 255) << 22) |
            (static_cast<unsigned long long>(t.ptab[rr][bq] >> 8) << 27);
    }
    for (int e = threadIdx.x; e < R * TB; e += blockDim.x) {
        const int r = e / TB, x = e % TB;
        const int code = t.pinv[r][x], role = code >> 7, pq = t.ptab[r][code & 127];
        t.part[r][x] = static_cast<unsigned char>((role ? (pq & 255) : (pq >> 8)) | (role << 7));
    }
    __syncthreads();
    const uint4* src = reinterpret_cast<const uint4*>(&t);
    uint4* dst = reinterpret_cast<uint4*>(out + mode);
    for (int e = threadIdx.x; e < static_cast<int>(sizeof(t) / 16); e += blockDim.x) dst[e] = src[e];
}

template <int TB>
__device__ __forceinline__ void solve_pair(const double* A, int64_t lda, const SolveTables<TB>* tabs,
                                           double* Qbuf, int* active, int nb, int round,
                                           const double* skip_tau_p, int max_inner, int mode, int pair) {
    // mode 0: all pairs of the 2b subproblem (2b-1 rounds of b rotations);
    // mode 1: only the pairs inside block I and inside block J (b-1 rounds);
    // mode 2: only the b^2 cross pairs (i in I, j in J) (b rounds).
    constexpr int B = TB / 2, LD = TB + 4, NP = TB / 2, RMAX = TB - 1;
    const int R = mode == 0 ? TB - 1 : (mode == 1 ? B - 1 : B);
    constexpr int MT = NP * NP;  // M threads
    constexpr int QW = solve_q_warps<TB>(), QR = TB / QW;
    constexpr int QT = 32 * QW;  // Q warps: lane l of warp h holds rows [h QR, (h+1) QR) of column l
    extern __shared__ double sm[];
    double* Mc = sm;             // current M
    double* Mn = Mc + TB * LD;   // next M (double buffer)
    double* Q = Mn + TB * LD;
    double* T = Q + TB * LD;
    (void)RMAX;
    __shared__ SolveTables<TB> st;  // inner schedule (see SolveTables)
    __shared__ double cs[RMAX][NP], sn[RMAX][NP];

    const int tid = threadIdx.x;
    // Role index (M threads, Q warps, then the lookahead warp). Making the
    // lookahead warp 0 instead (older warps are favoured by the schedulers)
    // measured no faster: 1361 vs 1311 cycles per inner round.
    const int rt = tid;
    const bool probe_round = pair == 0 && round == 5;
    const bool probe = probe_round && rt == MT + QT;
    long long t0 = SVDK_CLOCK();
    int I, J;
    circle_pair(nb, round, pair, I, J);
    // Everything the solve needs is fetched with all loads in flight at once:
    // the 32 x 32 block of A (<= 4 per thread) and this mode's precomputed
    // schedule tables (jacobi_tables_kernel, 16-byte loads).
    constexpr int NT = solve_threads<TB>();
    constexpr int PER = (TB * TB + NT - 1) / NT;
    {
        const uint4* src = reinterpret_cast<const uint4*>(tabs) + static_cast<size_t>(mode) *
                               (sizeof(SolveTables<TB>) / 16);
        uint4* dst = reinterpret_cast<uint4*>(&st);
        pdl_trigger();
        for (int e = tid; e < static_cast<int>(sizeof(SolveTables<TB>) / 16); e += NT) dst[e] = src[e];
    }
    pdl_wait();  // A (and the Q / active slots) of the previous round's update
    const double skip_tau = *skip_tau_p;  // written before the sweep (jacobi_start_kernel)
    bool big = false;
    {
        double xv[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = tid + k * NT;
            xv[k] = e < TB * TB ? __ldcg(&A[gidx(B, I, J, e % TB) + gidx(B, I, J, e / TB) * lda]) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = tid + k * NT;
            if (e < TB * TB) {
                const int i = e % TB, j = e / TB;
                Mc[i + j * LD] = xv[k];
                big |= (i != j) && fabs(xv[k]) > skip_tau;
            }
        }
    }
    const bool work = __syncthreads_or(big) != 0;
    auto& ptab = st.ptab;
    auto& pinv = st.pinv;
    long long t1 = SVDK_CLOCK();
    if (probe && work) {
        SVDK_PROBE_STORE(g_jprobe, 0, t0);
        SVDK_PROBE_STORE(g_jprobe, 1, t1);
    }
    if (work) {
        // Roles: MT "M threads" apply round rr to one 2x2 block each
        // (M <- R^T M R, double-buffered); the Q warps apply it to the rows of
        // Q; and the lookahead warp (lanes < NP) already evaluates round rr+1's
        // rotations: it recomputes, from M_rr and round rr's rotations, exactly
        // the three entries of M_rr+1 each new rotation needs (xform2x2's
        // operation order, same values as the M threads). The serial FP64
        // rotation chain then overlaps the round's update; a round costs one
        // block barrier plus the named-barrier gate behind the lookahead's reads.
        const int lane = rt - (MT + QT);
        auto rot_of = [&](int r, int i, const double* M) {  // initial round only
            const int code = ptab[r][i];
            const int p = code & 255, q = code >> 8;
            const double x = M[p + q * LD];
            double c = 1.0, s = 0.0;
            if (fabs(x) > skip_tau) rotation(M[p + p * LD], M[q + q * LD], x, c, s);
            cs[r][i] = c;
            sn[r][i] = s;
        };
        if (lane >= 0 && lane < NP) rot_of(0, lane, Mc);
        double qreg[QR];  // the Q warps' column slices (lane < TB)
        const int qrow0 = ((rt - MT) >> 5) * QR;
#pragma unroll
        for (int i = 0; i < QR; ++i) qreg[i] = (qrow0 + i == ((rt - MT) & 31)) ? 1.0 : 0.0;
        __syncthreads();
        const int total = max_inner * R;
        for (int it = 0; it < total; ++it) {
            const int rr = it % R;
            const bool pr = probe && it == 10;
            long long ta = (probe_round && it == 10) ? SVDK_CLOCK() : 0;
            if (rt < MT + QT) {
                if (rt < MT) {
                    const int bi = rt % NP, bj = rt / NP;
                    const int ci_code = ptab[rr][bi], cj_code = ptab[rr][bj];
                    const int pi = ci_code & 255, qi = ci_code >> 8;
                    const int pj = cj_code & 255, qj = cj_code >> 8;
                    double m00 = Mc[pi + pj * LD], m01 = Mc[pi + qj * LD];
                    double m10 = Mc[qi + pj * LD], m11 = Mc[qi + qj * LD];
                    xform2x2(m00, m01, m10, m11, cs[rr][bi], sn[rr][bi], cs[rr][bj], sn[rr][bj], bi == bj);
                    Mn[pi + pj * LD] = m00;
                    Mn[pi + qj * LD] = m01;
                    Mn[qi + pj * LD] = m10;
                    Mn[qi + qj * LD] = m11;
#ifdef SVDK_PROBES
                    if (probe_round && rt == 0 && it == 10) g_jprobe[9] = SVDK_CLOCK() - ta;
#endif
                } else {
                    // Q <- Q J: columns p, q of a rotation mix; partner columns are
                    // exchanged by warp shuffles (no shared-memory traffic)
                    const int l = (rt - MT) & 31;
                    const int code = pinv[rr][l & (TB - 1)];
                    const int j = code & 127, role = code >> 7;
                    const int pq = ptab[rr][j];
                    const int partner = role ? (pq & 255) : (pq >> 8);
                    // branch-free: a skipped pair has (c, s) = (1, 0)
                    const double c = cs[rr][j], b = role ? sn[rr][j] : -sn[rr][j];
#pragma unroll
                    for (int i = 0; i < QR; ++i) {
                        const double other = __shfl_sync(0xffffffffu, qreg[i], partner);
                        qreg[i] = fma(b, other, c * qreg[i]);
                    }
#ifdef SVDK_PROBES
                    if (probe_round && rt == MT && it == 10) {
                        double u;
                        asm volatile("add.f64 %0, %1, %2;" : "=d"(u) : "d"(qreg[0]), "d"(qreg[QR - 1]));
                        g_jprobe[10] = SVDK_CLOCK() - ta;
                        g_jprobe[13] = static_cast<long long>(u);
                    }
#endif
                }
            } else {
                // lookahead: rotation `lane` of round nr from M_{rr+1} entries
                const bool la = lane < NP && it + 1 < total;
                LookRead lr;
                if (la) lr = look_load<LD>(st, Mc, cs, sn, rr, lane, pr ? g_jprobe + 12 : nullptr, ta);
#ifdef SVDK_PROBES
                if (pr) {
                    double u;
                    asm volatile("add.f64 %0, %1, %2;" : "=d"(u) : "d"(lr.a00), "d"(lr.x11));
                    asm volatile("add.f64 %0, %0, %1;" : "+d"(u) : "d"(lr.cq));
                    g_jprobe[11] = SVDK_CLOCK() - ta;
                    g_jprobe[14] = static_cast<long long>(u);
                }
#endif
                if (la) {
                    long long t1 = pr ? SVDK_CLOCK() : 0;
                    double c, s;
                    look_finish(lr, skip_tau, c, s);
                    const int nr = (it + 1) % R;
                    cs[nr][lane] = c;
                    sn[nr][lane] = s;
                    if (pr) {
                        SVDK_PROBE_STORE(g_jprobe, 3, t1 - ta);
                        SVDK_PROBE_STORE(g_jprobe, 4, SVDK_CLOCK() - t1);
                    }
                }
            }
            long long tb = pr ? SVDK_CLOCK() : 0;
            __syncthreads();
            if (pr) {
                SVDK_PROBE_STORE(g_jprobe, 6, tb - ta);
                SVDK_PROBE_STORE(g_jprobe, 7, SVDK_CLOCK() - tb);
            }
            double* t = Mc;
            Mc = Mn;
            Mn = t;
        }
        if (rt >= MT && rt < MT + QT && ((rt - MT) & 31) < TB) {  // Q slices back to shared memory
            const int l = (rt - MT) & 31;
#pragma unroll
            for (int i = 0; i < QR; ++i) Q[(qrow0 + i) + l * LD] = qreg[i];
        }
        __syncthreads();
        if (probe) SVDK_PROBE_STORE(g_jprobe, 2, SVDK_CLOCK());
        // The product of ~TB * sweeps rotations drifts from orthogonality by a
        // few hundred ulps; one Newton-Schulz step Q <- Q (3I - Q^T Q) / 2
        // restores it to working precision so that A' = Q^T A Q is a
        // similarity to rounding (otherwise the spectrum drifts over sweeps).
        smem_mma<TB, true>(Q, Q, Mn);  // Mn <- Q^T Q
        __syncthreads();
        for (int e = tid; e < TB * TB; e += blockDim.x) {
            const int i = e % TB, j = e / TB;
            Mn[i + j * LD] = (i == j ? 1.5 : 0.0) - 0.5 * Mn[i + j * LD];
        }
        __syncthreads();
        smem_mma<TB, false>(Q, Mn, T);  // T <- Q (3I - Q^T Q) / 2
        __syncthreads();
        for (int e = tid; e < TB * TB; e += blockDim.x)
            Qbuf[static_cast<size_t>(pair) * TB * TB + e] = T[(e % TB) + (e / TB) * LD];
    }
    if (tid == 0) active[pair] = work ? 1 : 0;
    __syncthreads();  // shared memory is reused by the next pair / phase
}

// skip_tau is read from device memory (written by the sweep setup before the
// sweep graph runs), so one instantiated graph serves every eig_sym call.
template <int TB>
__global__ void __launch_bounds__(solve_threads<TB>())
    jacobi_pair_solve(const double* A, int64_t lda, const SolveTables<TB>* tabs, double* Qbuf,
                      int* active, int nb, int round, const double* skip_tau_p, int max_inner, int mode) {
    solve_pair<TB>(A, lda, tabs, Qbuf, active, nb, round, skip_tau_p, max_inner, mode, blockIdx.x);
}


// ---------------------------------------------------------------------------
// 1b. one-sided pair solve (2b = 32, the default for every n > 64)
// ---------------------------------------------------------------------------
// The same rotations in the same order as solve_pair, but the subproblem is
// never updated two-sidedly. The CTA keeps Q (starts at I) and W = M Q (starts
// at M) and applies every rotation as a COLUMN operation to both, so that the
// three numbers a rotation needs are dot products,
//     (Q^T M Q)_pp = q_p . w_p,   (Q^T M Q)_qq = q_q . w_q,   (Q^T M Q)_pq = q_p . w_q
// (the symmetric-eigenproblem form of Hestenes' one-sided method; M may be
// indefinite). Lane l of every warp owns column l, warp h the rows
// [h QR, (h+1) QR) of both matrices: 2 QR registers per lane, the partner
// column arrives by warp shuffles, and the only cross-warp traffic of an inner
// round is the QW partial sums per dot product through shared memory (summed
// in warp order by every lane, so all warps form bit-identical (c, s)) behind
// ONE block barrier. The serial chain of a round is
//     shuffle -> partial dots -> STS | barrier | LDS -> sum -> rotation -> apply
// with QW warps instead of 13, no M threads, no lookahead and ~100 instead of
// ~390 shared-memory wavefronts (solve_pair: ~1230 cycles per inner round,
// §3.2 of DESIGN.md). a_pq is formed with an absolute error of a few
// eps ||M||, the same floor the DMMA similarity Q^T A Q of the update kernels
// has; the convergence test stays on the explicitly updated A.
// 1 / sqrt(x) for normal x > 0 from the hardware seed (rsqrt.approx.ftz.f64, ~2^-22) and
// one third-order step y (1 + e/2 + 3e^2/8), e = 1 - x y^2: a 4-DFMA chain behind the
// MUFU instead of rsqrt()'s ~100 cycles (its special-case handling is not needed:
// eig_sym prescales so that d^2 + e^2 stays normal).
__device__ __forceinline__ double rsqrt_seed(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double rsqrt_refine(double x, double y0) {
    const double t = x * y0;
    const double e = fma(-t, y0, 1.0);
    return fma(y0 * e, fma(0.375, e, 0.5), y0);
}
// rotation() with the second square root's seed formed speculatively from the
// first one's seed, so the two refinements are the only dependent DFMA chains
// (~140 instead of ~210 cycles; same formulas, results equal to a few ulps).
__device__ __forceinline__ void rotation_fast(double app, double aqq, double apq, double& c, double& s) {
    const double d = aqq - app, e = 2.0 * apq, e2 = e * e, ad = fabs(d);
    const double r2 = fma(d, d, e2);
    const double y0 = rsqrt_seed(r2);
    const double Dt = ad + r2 * y0;
    const double z0 = rsqrt_seed(fma(Dt, Dt, e2));  // seed of the second root, off the precise chain
    const double D = ad + r2 * rsqrt_refine(r2, y0);  // |d| + sqrt(d^2 + e^2)
    const double inv = rsqrt_refine(fma(D, D, e2), z0);
    c = D * inv;
    s = (d > 0.0 ? e : (d < 0.0 ? -e : fabs(e))) * inv;  // tau = +-0 -> t = +1
}

__device__ __forceinline__ double4 ld_cg4(const double* p);
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d);

// `total` inner rounds of the one-sided solve on this lane's column slabs
// (QR rows of Q and of W = M Q) for one 32-column subproblem shared by QW
// warps that meet at named barrier `bar` (see jacobi_pair_solve_os).
// sched[r][lane] = partner lane | role << 7 for the R rounds of the schedule;
// pd / px = [2][QW][32] partial-sum buffers of this subproblem. Returns
// whether this lane applied any rotation.
template <int QR, int QW, bool FAST>
__device__ __forceinline__ bool os_rounds(double (&qreg)[QR], double (&wreg)[QR],
                                          const unsigned char (*sched)[32], int R, int total,
                                          double (*pd)[QW][32], double (*px)[QW][32], int w, int lane,
                                          int bar, double skip_tau) {
    int code = sched[0][lane], rr = 0;
    bool rotated = false;
    for (int it = 0; it < total; ++it) {
        const int partner = code & 31, role = code >> 7, buf = it & 1;
        rr = rr + 1 == R ? 0 : rr + 1;
        code = sched[rr][lane];  // next round's pairing, off the chain
        double oq[QR], ow[QR];
#pragma unroll
        for (int i = 0; i < QR; ++i) {
            oq[i] = __shfl_sync(0xffffffffu, qreg[i], partner);
            ow[i] = __shfl_sync(0xffffffffu, wreg[i], partner);
        }
        // partial dots over this warp's rows: own diagonal and (role p) q_p . w_q
        double d0 = qreg[0] * wreg[0], d1 = qreg[1] * wreg[1];
        double x0 = qreg[0] * ow[0], x1 = qreg[1] * ow[1];
#pragma unroll
        for (int i = 2; i < QR; i += 2) {
            d0 = fma(qreg[i], wreg[i], d0);
            d1 = fma(qreg[i + 1], wreg[i + 1], d1);
            x0 = fma(qreg[i], ow[i], x0);
            x1 = fma(qreg[i + 1], ow[i + 1], x1);
        }
        pd[buf][w][lane] = d0 + d1;
        px[buf][w][lane] = x0 + x1;
        named_bar(bar, 32 * QW);
        const int pl = role ? partner : lane;  // the pair's p column
        double ds = 0.0, dp = 0.0, xs = 0.0;
#pragma unroll
        for (int h = 0; h < QW; h += 2) {  // fixed order: identical bits in every warp
            ds += pd[buf][h][lane] + pd[buf][h + 1][lane];
            dp += pd[buf][h][partner] + pd[buf][h + 1][partner];
            xs += px[buf][h][pl] + px[buf][h + 1][pl];
        }
        double c = 1.0, s = 0.0;
        if (fabs(xs) > skip_tau) {
            rotated = true;
            if (FAST)
                rotation_fast(role ? dp : ds, role ? ds : dp, xs, c, s);
            else
                rotation(role ? dp : ds, role ? ds : dp, xs, c, s);
        }
        const double b = role ? s : -s;  // column p: c q_p - s q_q; column q: s q_p + c q_q
#pragma unroll
        for (int i = 0; i < QR; ++i) {
            qreg[i] = fma(b, oq[i], c * qreg[i]);
            wreg[i] = fma(b, ow[i], c * wreg[i]);
        }
    }
    return rotated;
}

template <int QW, bool NS, bool FAST>
__global__ void __launch_bounds__(32 * QW)
    jacobi_pair_solve_os(const double* A, int64_t lda, const SolveTables<32>* tabs, double* Qbuf,
                         int* active, int nb, int round, const double* skip_tau_p, int max_inner, int mode) {
    constexpr int TB = 32, B = 16, LD = TB + 4, QR = TB / QW;
    static_assert(QR % 4 == 0 && QR <= 16, "row slabs are 32-byte vectors inside one 16-index block");
    __shared__ __align__(16) unsigned char sched[TB - 1][TB];
    __shared__ double pd[2][QW][TB], px[2][QW][TB];
    __shared__ double Qs[TB * LD], Ms[TB * LD], Ts[TB * LD];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, pair = blockIdx.x;
    const int R = mode == 0 ? TB - 1 : (mode == 1 ? B - 1 : B);
    const bool probe = pair == 0 && round == 5 && tid == 0;
    const long long t0 = SVDK_CLOCK();
    int I, J;
    circle_pair(nb, round, pair, I, J);
    {
        const uint4* src = reinterpret_cast<const uint4*>(&tabs[mode].part[0][0]);
        uint4* dst = reinterpret_cast<uint4*>(&sched[0][0]);
        pdl_trigger();
        for (int e = tid; e < static_cast<int>(sizeof(sched) / 16); e += 32 * QW) dst[e] = src[e];
    }
    pdl_wait();  // A (and the Q / active slots) of the previous round's update
    const double skip_tau = *skip_tau_p;
    const int row0 = w * QR;
    double wreg[QR], qreg[QR];
    bool big = false;
    {
        const double* col = A + gidx(B, I, J, row0) + gidx(B, I, J, lane) * lda;
#pragma unroll
        for (int v = 0; v < QR / 4; ++v) {
            const double4 x = ld_cg4(col + 4 * v);
            wreg[4 * v] = x.x; wreg[4 * v + 1] = x.y; wreg[4 * v + 2] = x.z; wreg[4 * v + 3] = x.w;
        }
#pragma unroll
        for (int i = 0; i < QR; ++i) {
            big |= (row0 + i != lane) && fabs(wreg[i]) > skip_tau;
            qreg[i] = (row0 + i == lane) ? 1.0 : 0.0;
        }
    }
    const bool work = __syncthreads_or(big) != 0;
    if (probe && work) {
        SVDK_PROBE_STORE(g_jprobe, 0, t0);
        SVDK_PROBE_STORE(g_jprobe, 1, SVDK_CLOCK());
    }
    if (work) {
        const int total = max_inner * R;
        os_rounds<QR, QW, FAST>(qreg, wreg, sched, R, total, pd, px, w, lane, 0, skip_tau);
        if (probe) SVDK_PROBE_STORE(g_jprobe, 2, SVDK_CLOCK());
        if (NS) {
#pragma unroll
            for (int i = 0; i < QR; ++i) Qs[(row0 + i) + lane * LD] = qreg[i];
            __syncthreads();
            // Newton-Schulz step Q <- Q (3I - Q^T Q) / 2 (see solve_pair)
            smem_mma<TB, true>(Qs, Qs, Ms);
            __syncthreads();
            for (int e = tid; e < TB * TB; e += 32 * QW) {
                const int i = e % TB, j = e / TB;
                Ms[i + j * LD] = (i == j ? 1.5 : 0.0) - 0.5 * Ms[i + j * LD];
            }
            __syncthreads();
            smem_mma<TB, false>(Qs, Ms, Ts);
            __syncthreads();
            for (int e = tid; e < TB * TB; e += 32 * QW)
                Qbuf[static_cast<size_t>(pair) * TB * TB + e] = Ts[(e % TB) + (e / TB) * LD];
        } else {
            // A rotation with c^2 + s^2 = 1 + delta scales its two columns and keeps
            // them orthogonal (J^T J = (1 + delta) I), so the accumulated Q departs
            // from orthogonality in its column norms only (plus unbiased rounding of
            // the column operations): one Newton step on each column's norm,
            // q <- q (3 - |q|^2) / 2, replaces the Newton-Schulz products.
            double n0 = qreg[0] * qreg[0], n1 = qreg[1] * qreg[1];
#pragma unroll
            for (int i = 2; i < QR; i += 2) {
                n0 = fma(qreg[i], qreg[i], n0);
                n1 = fma(qreg[i + 1], qreg[i + 1], n1);
            }
            const int buf = total & 1;
            pd[buf][w][lane] = n0 + n1;
            __syncthreads();
            double nn = 0.0;
#pragma unroll
            for (int h = 0; h < QW; h += 2) nn += pd[buf][h][lane] + pd[buf][h + 1][lane];
            const double f = fma(-0.5, nn, 1.5);
            double* out = Qbuf + static_cast<size_t>(pair) * TB * TB + row0 + lane * TB;
#pragma unroll
            for (int v = 0; v < QR / 4; ++v)
                st4(out + 4 * v, f * qreg[4 * v], f * qreg[4 * v + 1], f * qreg[4 * v + 2], f * qreg[4 * v + 3]);
        }
    }
    if (tid == 0) active[pair] = work ? 1 : 0;
    if (probe && work) SVDK_PROBE_STORE(g_jprobe, 3, SVDK_CLOCK());
}



// ---------------------------------------------------------------------------
// 2. the round's similarity on A, and its accumulation into V
// ---------------------------------------------------------------------------
// jacobi_update_a: one CTA per pair block (p <= q):
//   A[IJ_p, IJ_q] <- Q_p^T A[IJ_p, IJ_q] Q_q   (mirror written from the same
//   values so A stays exactly symmetric; diagonal pair blocks symmetrised).
template <int TB>
__global__ void __launch_bounds__(256)
    jacobi_update_a(double* A, int64_t lda, const double* Qbuf, const int* active, int nb,
                    int round) {
    constexpr int B = TB / 2, LD = TB + 4;
    extern __shared__ double sm[];
    double* X = sm;
    double* Qa = X + TB * LD;
    double* Qb = Qa + TB * LD;
    double* T = Qb + TB * LD;
    const int tid = threadIdx.x;
    const int u = blockIdx.x;
    // (p <= q) from u, column-wise upper enumeration
    int q = static_cast<int>((sqrt(8.0 * u + 1.0) - 1.0) * 0.5);
    while ((q + 1) * (q + 2) / 2 <= u) ++q;
    while (q * (q + 1) / 2 > u) --q;
    const int p = u - q * (q + 1) / 2;
    const int ap = active[p], aq = active[q];
    if (!(ap | aq)) return;  // both rotations are the identity
    int Ip, Jp, Iq, Jq;
    circle_pair(nb, round, p, Ip, Jp);
    circle_pair(nb, round, q, Iq, Jq);
    const double* qa = Qbuf + static_cast<size_t>(p) * TB * TB;
    const double* qb = Qbuf + static_cast<size_t>(q) * TB * TB;
    for (int e = tid; e < TB * TB; e += blockDim.x) {
        const int i = e % TB, j = e / TB;
        X[i + j * LD] = A[gidx(B, Ip, Jp, i) + gidx(B, Iq, Jq, j) * lda];
        Qa[i + j * LD] = ap ? qa[e] : (i == j ? 1.0 : 0.0);
        Qb[i + j * LD] = aq ? qb[e] : (i == j ? 1.0 : 0.0);
    }
    __syncthreads();
    smem_mma<TB, false>(X, Qb, T);  // T = X Q_q
    __syncthreads();
    smem_mma<TB, true>(Qa, T, X);   // X = Q_p^T T
    __syncthreads();
    if (p == q) {  // diagonal pair block: write the exactly symmetric part
        for (int e = tid; e < TB * TB; e += blockDim.x) {
            const int i = e % TB, j = e / TB;
            A[gidx(B, Ip, Jp, i) + gidx(B, Ip, Jp, j) * lda] = 0.5 * (X[i + j * LD] + X[j + i * LD]);
        }
        return;
    }
    for (int e = tid; e < TB * TB; e += blockDim.x) {
        const int i = e % TB, j = e / TB;
        A[gidx(B, Ip, Jp, i) + gidx(B, Iq, Jq, j) * lda] = X[i + j * LD];
    }
    for (int e = tid; e < TB * TB; e += blockDim.x) {
        const int j = e % TB, i = e / TB;  // consecutive threads walk rows of the mirror
        A[gidx(B, Iq, Jq, j) + gidx(B, Ip, Jp, i) * lda] = X[i + j * LD];
    }
}

// jacobi_update_v: one CTA per (row tile, pair q): V[rows, IJ_q] <- V[rows, IJ_q] Q_q.
// V never feeds back into the iteration, so these launches run on a side
// stream, overlapped with the next rounds' latency-bound pair solves.
template <int TB>
__global__ void __launch_bounds__(256)
    jacobi_update_v(double* V, int64_t ldv, const double* Qbuf, const int* active, int nb,
                    int round) {
    constexpr int B = TB / 2, LD = TB + 4;
    extern __shared__ double sm[];
    double* X = sm;
    double* Qb = X + TB * LD;
    double* T = Qb + TB * LD;
    const int tid = threadIdx.x;
    const int k = nb / 2;
    const int q = blockIdx.x % k;
    if (!active[q]) return;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x / k) * TB;
    int Iq, Jq;
    circle_pair(nb, round, q, Iq, Jq);
    const double* qb = Qbuf + static_cast<size_t>(q) * TB * TB;
    for (int e = tid; e < TB * TB; e += blockDim.x) {
        const int i = e % TB, j = e / TB;
        X[i + j * LD] = V[r0 + i + gidx(B, Iq, Jq, j) * ldv];
        Qb[i + j * LD] = qb[e];
    }
    __syncthreads();
    smem_mma<TB, false>(X, Qb, T);
    __syncthreads();
    for (int e = tid; e < TB * TB; e += blockDim.x) {
        const int i = e % TB, j = e / TB;
        V[r0 + i + gidx(B, Iq, Jq, j) * ldv] = T[i + j * LD];
    }
}

// Register-resident variants for 2b = 32 (used for every n > 64). One WARP
// owns one 32 x 32 block and never touches shared memory: the operands are
// loaded straight into m8n8k4 fragments (A rows: 8 consecutive doubles of a
// column per lane quad -> full 32 B sectors), the intermediate U = Q_p^T X of
// the two-sided product is re-laid from accumulator to A-fragment form with
// quad shuffles, and results are stored from the accumulators. No barriers,
// and every warp keeps its whole 8 KB tile in flight, so the kernels run at
// HBM rate instead of the load -> sync -> compute -> sync chain of the
// shared-memory versions above.
//
// Fragment maps (mma.m8n8k4.row.col, lane = 4 r + kq):
//   A[m][k]: A[r][kq]     B[k][n]: B[kq][r]     C: C[r][2 kq], C[r][2 kq + 1]
__device__ __forceinline__ double q_frag(const double* Qp, bool act, int k, int n) {
    // Q[k][n] of a column-major 32 x 32 rotation, identity when inactive
    return act ? __ldcg(&Qp[k + n * 32]) : (k == n ? 1.0 : 0.0);
}

// 32-byte global accesses (one full sector; LDG/STG.E.ENL2.256 on sm_100)
__device__ __forceinline__ double4 ld_cg4(const double* p) {
    double4 v;
    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

constexpr int UPD_WARPS = 4;

// A[IJ_p, IJ_q] <- Q_p^T A[IJ_p, IJ_q] Q_q for one (p <= q) per warp; the
// mirror block gets the same values (exact symmetry); a diagonal pair block
// copies its upper triangle to the lower one.
__device__ __forceinline__ void upd_a_unit(double* A, int64_t lda, const double* Qbuf,
                                           const int* active, int nb, int round, int u) {
    constexpr int B = 16;
    const int lane = threadIdx.x & 31, r = lane >> 2, kq = lane & 3;
    const int k = nb / 2;
    pdl_trigger();
    pdl_wait();
    if (u >= k * (k + 1) / 2) return;
    int q = static_cast<int>((sqrt(8.0 * u + 1.0) - 1.0) * 0.5);
    while ((q + 1) * (q + 2) / 2 <= u) ++q;
    while (q * (q + 1) / 2 > u) --q;
    const int p = u - q * (q + 1) / 2;
    const bool ap = __ldcg(&active[p]) != 0, aq = __ldcg(&active[q]) != 0;
    if (!(ap | aq)) return;  // both rotations are the identity
    int Ip, Jp, Iq, Jq;
    circle_pair(nb, round, p, Ip, Jp);
    circle_pair(nb, round, q, Iq, Jq);
    const double* Qa = Qbuf + static_cast<size_t>(p) * 1024;
    const double* Qb = Qbuf + static_cast<size_t>(q) * 1024;
    // step 1: U = Q_p^T X. A-frags (Q_p^T)[m][k] = Q_p[k][m]; B-frags X[k][n].
    double xa[8][4], xb[8][4];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const int64_t row = gidx(B, Ip, Jp, 4 * s + kq);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            xb[s][t] = __ldcg(&A[row + gidx(B, Iq, Jq, 8 * t + r) * lda]);
            xa[s][t] = q_frag(Qa, ap, 4 * s + kq, 8 * t + r);
        }
    }
    double acc[4][4][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int t = 0; t < 4; ++t) dmma(acc[m][t][0], acc[m][t][1], xa[s][m], xb[s][t]);
    // step 2: X' = U Q_q. U[8m + r][4s + kq] lives in lane (r, 2(s&1) + kq/2),
    // register acc[m][s/2][kq&1].
    double qb[8][4];
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int t = 0; t < 4; ++t) qb[s][t] = q_frag(Qb, aq, 4 * s + kq, 8 * t + r);
    double out[4][4][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int t = 0; t < 4; ++t) out[m][t][0] = out[m][t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const int src = (lane & ~3) | (2 * (s & 1) + (kq >> 1));
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const double v0 = __shfl_sync(0xffffffffu, acc[m][s >> 1][0], src);
            const double v1 = __shfl_sync(0xffffffffu, acc[m][s >> 1][1], src);
            const double a = (kq & 1) ? v1 : v0;
#pragma unroll
            for (int t = 0; t < 4; ++t) dmma(out[m][t][0], out[m][t][1], a, qb[s][t]);
        }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int li = 8 * m + r;
        const int64_t gi = gidx(B, Ip, Jp, li);
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int lj = 8 * t + 2 * kq + i;
                const int64_t gj = gidx(B, Iq, Jq, lj);
                if (p == q && li > lj) continue;
                A[gi + gj * lda] = out[m][t][i];
                A[gj + gi * lda] = out[m][t][i];
            }
    }
}

// The same unit with both contractions re-indexed so that no data crosses
// lanes and every operand load is a vector load (one warp per unit):
//   step 1, U = Q_p^T X: k-step s takes contraction index
//     k1(s, kq) = 16 (s >> 2) + 4 kq + (s & 3)
//   so lane (r, kq) needs rows 16h + 4kq .. +3 of a column of Q_p and of X for
//   the four k-steps of half h: one 32-byte load each (8 + 8 instead of
//   32 + 32 scalar loads);
//   step 2, X' = U Q_q: k-step s takes k2(s, kq) = 8 (s >> 1) + 2 kq + (s & 1),
//   which is exactly the column of U that lane (r, kq) already holds in
//   accumulator acc[m][s >> 1][s & 1] (C layout C[r][2 kq + i]), so the 64
//   quad shuffles of upd_a_unit disappear; Q_q is read as 16-byte row pairs.
// The contraction order differs from upd_a_unit (a permutation of k), so the
// results differ from it by rounding only. The mirror block is written with
// 16-byte stores (rows 2kq, 2kq+1 of a column).
__device__ __forceinline__ double2 ld_cg2(const double* p) {
    double2 v;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void st2(double* p, double a, double b) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

// MS warps share a unit (MS = 1, 2, 4): warp `part` forms the rows
// [32 part / MS, 32 (part + 1) / MS) of X' (its rows of U stay in its own
// accumulators) and reads all of X and Q_q; the warps of a CTA meet at a
// barrier between the last read of X and the first store.
// !INPLACE (solve-ahead ping-pong, Aout != A): every block is written, also
// where both rotations are the identity, and the warps of a unit need no
// barrier between their reads and stores.
template <int MS, bool INPLACE = true>
__device__ __forceinline__ void upd_a_unit_vec(const double* A, double* Aout, int64_t lda, const double* Qbuf,
                                               const int* active, int nb, int round, int u, int part) {
    constexpr int B = 16, MW = 4 / MS;  // m-tiles (8 rows each) per warp
    const int lane = threadIdx.x & 31, r = lane >> 2, kq = lane & 3;
    const int k = nb / 2;
    pdl_trigger();
    pdl_wait();  // Q_p, Q_q and the active flags of this round's solve
    bool live = u < k * (k + 1) / 2;
    int p = 0, q = 0;
    if (live) {
        q = static_cast<int>((sqrt(8.0 * u + 1.0) - 1.0) * 0.5);
        while ((q + 1) * (q + 2) / 2 <= u) ++q;
        while (q * (q + 1) / 2 > u) --q;
        p = u - q * (q + 1) / 2;
    }
    const bool ap = live && __ldcg(&active[p]) != 0, aq = live && __ldcg(&active[q]) != 0;
    live = live && ((ap | aq) || !INPLACE);  // in place, both rotations the identity: nothing to do
    int Ip, Jp, Iq, Jq;
    circle_pair(nb, round, p, Ip, Jp);
    circle_pair(nb, round, q, Iq, Jq);
    const double* Qa = Qbuf + static_cast<size_t>(p) * 1024;
    const double* Qb = Qbuf + static_cast<size_t>(q) * 1024;
    const int m0 = part * MW;
    if (!INPLACE && MS == 2 && live && !(ap | aq)) {
        // ping-pong and both rotations the identity (late sweeps, the polish sweep): this half of the
        // block and its mirror are copied, no DMMA work
        const int64_t gi0 = static_cast<int64_t>(part ? Jp : Ip) * B + 4 * kq;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int64_t gc = gidx(B, Iq, Jq, 8 * t + r);
            const double4 v = ld_cg4(A + gi0 + gc * lda);
            st4(Aout + gi0 + gc * lda, v.x, v.y, v.z, v.w);
            if (p != q) {
                Aout[gc + gi0 * lda] = v.x;
                Aout[gc + (gi0 + 1) * lda] = v.y;
                Aout[gc + (gi0 + 2) * lda] = v.z;
                Aout[gc + (gi0 + 3) * lda] = v.w;
            }
        }
        return;
    }
    double out[MW][4][2];
    if (live) {
        // global row of local index 16h + 4kq (h = 0: block I_p, 1: J_p) and
        // global column of local index 8t + r
        const int64_t rowh[2] = {static_cast<int64_t>(Ip) * B + 4 * kq, static_cast<int64_t>(Jp) * B + 4 * kq};
        int64_t colt[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) colt[t] = gidx(B, Iq, Jq, 8 * t + r);
        double4 xv[2][4], qa[2][MW];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int t = 0; t < 4; ++t) xv[h][t] = ld_cg4(A + rowh[h] + colt[t] * lda);
#pragma unroll
            for (int m = 0; m < MW; ++m) {
                // Q_p[16h + 4kq + j][8(m0 + m) + r]; identity when inactive
                const int k0 = 16 * h + 4 * kq, c = 8 * (m0 + m) + r;
                // the slot is read beside the active flag, not behind it (always allocated)
                qa[h][m] = ld_cg4(Qa + k0 + c * 32);
                if (!ap) qa[h][m] = make_double4(k0 == c, k0 + 1 == c, k0 + 2 == c, k0 + 3 == c);
            }
        }
        double2 qb[4][4];  // Q_q[8a + 2kq + {0,1}][8t + r]
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int k0 = 8 * a + 2 * kq, c = 8 * t + r;
                qb[a][t] = ld_cg2(Qb + k0 + c * 32);
                if (!aq) qb[a][t] = make_double2(k0 == c, k0 + 1 == c);
            }
        double acc[MW][4][2];
#pragma unroll
        for (int m = 0; m < MW; ++m)
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int h = s >> 2, j = s & 3;
#pragma unroll
            for (int m = 0; m < MW; ++m) {
                const double4 av = qa[h][m];
                const double a = j == 0 ? av.x : (j == 1 ? av.y : (j == 2 ? av.z : av.w));
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const double4 bv = xv[h][t];
                    const double b = j == 0 ? bv.x : (j == 1 ? bv.y : (j == 2 ? bv.z : bv.w));
                    dmma(acc[m][t][0], acc[m][t][1], a, b);
                }
            }
        }
#pragma unroll
        for (int m = 0; m < MW; ++m)
#pragma unroll
            for (int t = 0; t < 4; ++t) out[m][t][0] = out[m][t][1] = 0.0;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int a2 = s >> 1, i2 = s & 1;
#pragma unroll
            for (int m = 0; m < MW; ++m)
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    dmma(out[m][t][0], out[m][t][1], acc[m][a2][i2], i2 ? qb[a2][t].y : qb[a2][t].x);
        }
    }
    if (MS > 1 && INPLACE) __syncthreads();  // every warp of the CTA has read its X
    if (!live) return;
    if (p == q) {  // diagonal pair block: upper triangle and its mirror, scalar
#pragma unroll
        for (int m = 0; m < MW; ++m) {
            const int li = 8 * (m0 + m) + r;
            const int64_t gi = gidx(B, Ip, Jp, li);
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int lj = 8 * t + 2 * kq + i;
                    if (li > lj) continue;
                    const int64_t gj = gidx(B, Iq, Jq, lj);
                    Aout[gi + gj * lda] = out[m][t][i];
                    Aout[gj + gi * lda] = out[m][t][i];
                }
        }
        return;
    }
#pragma unroll
    for (int m = 0; m < MW; ++m) {
        const int64_t gi = gidx(B, Ip, Jp, 8 * (m0 + m) + r);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int64_t gj = gidx(B, Iq, Jq, 8 * t + 2 * kq);  // and gj + 1 (same 16-index block)
            Aout[gi + gj * lda] = out[m][t][0];
            Aout[gi + (gj + 1) * lda] = out[m][t][1];
            st2(Aout + gj + gi * lda, out[m][t][0], out[m][t][1]);
        }
    }
}

template <int MS>
__global__ void __launch_bounds__(UPD_WARPS * 32)
    jacobi_update_a_vec(const double* A, double* Aout, int64_t lda, const double* Qbuf, const int* active,
                        int nb, int round) {
    const int w = threadIdx.x >> 5;
    upd_a_unit_vec<MS>(A, Aout, lda, Qbuf, active, nb, round, blockIdx.x * (UPD_WARPS / MS) + w / MS, w % MS);
}

// The same update split over the four warps of a CTA (one unit per CTA):
// warp w4 produces rows [8 w4, 8 w4 + 8) of Q_p^T X Q_q. Its rows of
// U = Q_p^T X stay in its own accumulators, so no data crosses warps; each
// warp reads all of X and Q_q (L2-resident) and issues 64 instead of 256
// DMMAs, so a round's update takes the latency of a quarter of the work. The
// CTA meets at a barrier between the last read of X and the first store
// (every warp reads all of X and writes a quarter of it). Same accumulation
// order per output entry as upd_a_unit: bit-identical results. Used for
// n <= 768, where a round is a short latency chain (solve -> update -> solve).
__global__ void __launch_bounds__(128)
    jacobi_update_a_q4(double* A, int64_t lda, const double* Qbuf, const int* active, int nb, int round) {
    constexpr int B = 16;
    const int lane = threadIdx.x & 31, r = lane >> 2, kq = lane & 3, w4 = threadIdx.x >> 5;
    const int u = blockIdx.x;
    pdl_trigger();
    pdl_wait();
    int q = static_cast<int>((sqrt(8.0 * u + 1.0) - 1.0) * 0.5);
    while ((q + 1) * (q + 2) / 2 <= u) ++q;
    while (q * (q + 1) / 2 > u) --q;
    const int p = u - q * (q + 1) / 2;
    const bool ap = __ldcg(&active[p]) != 0, aq = __ldcg(&active[q]) != 0;
    if (!(ap | aq)) return;
    int Ip, Jp, Iq, Jq;
    circle_pair(nb, round, p, Ip, Jp);
    circle_pair(nb, round, q, Iq, Jq);
    const double* Qa = Qbuf + static_cast<size_t>(p) * 1024;
    const double* Qb = Qbuf + static_cast<size_t>(q) * 1024;
    double xa[8], xb[8][4], qb[8][4];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const int64_t row = gidx(B, Ip, Jp, 4 * s + kq);
        xa[s] = q_frag(Qa, ap, 4 * s + kq, 8 * w4 + r);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            xb[s][t] = __ldcg(&A[row + gidx(B, Iq, Jq, 8 * t + r) * lda]);
            qb[s][t] = q_frag(Qb, aq, 4 * s + kq, 8 * t + r);
        }
    }
    double acc[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int t = 0; t < 4; ++t) dmma(acc[t][0], acc[t][1], xa[s], xb[s][t]);
    double out[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) out[t][0] = out[t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const int src = (lane & ~3) | (2 * (s & 1) + (kq >> 1));
        const double v0 = __shfl_sync(0xffffffffu, acc[s >> 1][0], src);
        const double v1 = __shfl_sync(0xffffffffu, acc[s >> 1][1], src);
        const double a = (kq & 1) ? v1 : v0;
#pragma unroll
        for (int t = 0; t < 4; ++t) dmma(out[t][0], out[t][1], a, qb[s][t]);
    }
    __syncthreads();  // all of X has been read by every warp
    const int li = 8 * w4 + r;
    const int64_t gi = gidx(B, Ip, Jp, li);
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int lj = 8 * t + 2 * kq + i;
            const int64_t gj = gidx(B, Iq, Jq, lj);
            if (p == q && li > lj) continue;
            A[gi + gj * lda] = out[t][i];
            A[gj + gi * lda] = out[t][i];
        }
}

// V[rows, IJ_q] <- V[rows, IJ_q] Q_q; one warp per (pair q, VT_ROWS-row chunk).
// Rows inside a 32-row tile are permuted so that m8n8k4 row r of m-tile m is
// tile row 4r + m (each output row depends only on its own input row): lane
// (r, kq) then owns 4 CONSECUTIVE rows of a column, and every access is one
// 32-byte load/store (8 + 8 per tile instead of 32 + 32 scattered 8-byte
// ones). Q_q's fragments are loaded once per warp; the next tile's loads are
// in flight while the current tile's DMMAs run.
constexpr int VT_ROWS = 128;

__device__ __forceinline__ void upd_v_unit(double* V, int64_t ldv, int64_t n_rows,
                                           const double* Qbuf, const int* active, int nb, int round,
                                           int64_t u, int vt_rows = VT_ROWS) {
    constexpr int B = 16;
    const int lane = threadIdx.x & 31, r = lane >> 2, kq = lane & 3;
    const int k = nb / 2;
    const int q = static_cast<int>(u % k);
    const int64_t row_begin = (u / k) * vt_rows;
    if (row_begin >= n_rows || !__ldcg(&active[q])) return;
    const int64_t row_end = min(n_rows, row_begin + vt_rows);
    int Iq, Jq;
    circle_pair(nb, round, q, Iq, Jq);
    const double* Qb = Qbuf + static_cast<size_t>(q) * 1024;
    // The contraction index of k-step s is k(s, kq) = 16 (s >> 2) + 4 kq + (s & 3) (a permutation of
    // 0..31, the same in both operands), so a lane's Q_q fragments of four k-steps are four consecutive
    // rows of one column: 8 32-byte loads instead of 32 8-byte ones.
    double qb[8][4];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const double4 q4 = ld_cg4(Qb + 16 * h + 4 * kq + (8 * t + r) * 32);
            qb[4 * h][t] = q4.x; qb[4 * h + 1][t] = q4.y; qb[4 * h + 2][t] = q4.z; qb[4 * h + 3][t] = q4.w;
        }
    double* vb = V + 4 * r;
    int64_t vcol[8];  // column of V for k-step s
#pragma unroll
    for (int s = 0; s < 8; ++s) vcol[s] = gidx(B, Iq, Jq, 16 * (s >> 2) + 4 * kq + (s & 3)) * ldv;
    double4 va[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) va[s] = ld_cg4(vb + row_begin + vcol[s]);
    for (int64_t row0 = row_begin; row0 < row_end; row0 += 32) {
        const bool more = row0 + 32 < row_end;
        double4 vn[8];
        if (more) {
#pragma unroll
            for (int s = 0; s < 8; ++s) vn[s] = ld_cg4(vb + row0 + 32 + vcol[s]);
        }
        double acc[4][4][2];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const double am[4] = {va[s].x, va[s].y, va[s].z, va[s].w};
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int t = 0; t < 4; ++t) dmma(acc[m][t][0], acc[m][t][1], am[m], qb[s][t]);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int i = 0; i < 2; ++i)
                st4(vb + row0 + gidx(B, Iq, Jq, 8 * t + 2 * kq + i) * ldv, acc[0][t][i], acc[1][t][i],
                    acc[2][t][i], acc[3][t][i]);
        if (more) {
#pragma unroll
            for (int s = 0; s < 8; ++s) va[s] = vn[s];
        }
    }
}

__global__ void __launch_bounds__(UPD_WARPS * 32)
    jacobi_update_a_reg(double* A, int64_t lda, const double* Qbuf, const int* active, int nb,
                        int round) {
    upd_a_unit(A, lda, Qbuf, active, nb, round, blockIdx.x * UPD_WARPS + (threadIdx.x >> 5));
}

__global__ void __launch_bounds__(UPD_WARPS * 32)
    jacobi_update_v_reg(double* V, int64_t ldv, int64_t n_rows, const double* Qbuf,
                        const int* active, int nb, int round) {
    upd_v_unit(V, ldv, n_rows, Qbuf, active, nb, round,
               static_cast<int64_t>(blockIdx.x) * UPD_WARPS + (threadIdx.x >> 5));
}

// ---------------------------------------------------------------------------
// 2b. fused round kernel (solve-ahead), n_pad <= kAheadMaxN
// ---------------------------------------------------------------------------
// For small and medium n a round is a latency chain, solve -> A update ->
// solve. Here the pair solve of round j does not wait for round j-1's A
// update: it reads A_{j-2} (the matrix BEFORE round j-1's similarity, the
// other half of a ping-pong pair) and round j-1's rotations and forms its own
// 32 x 32 subproblem
//     M = T^T X T,   X = A_{j-2}[P, P] (64 x 64),   T = diag(T_I, T_J) (64 x 32),
// where block I sat in round j-1's pair p_I (T_I = the 16 columns of Q_{p_I}
// that belong to I), block J in p_J, and P = the four blocks of p_I and p_J.
// One kernel per round then holds three roles, all depending only on the
// previous kernel (one programmatic dependent launch chain on one stream):
//   CTAs [0, n_solve)            solve_j          (A_{j-2}, Q_{j-1} -> Q_j)
//   CTAs [.., + n_upd_a)         A update j-1     (A_{j-2}, Q_{j-1} -> A_{j-1}, other buffer)
//   CTAs [.., + n_upd_v)         V update j-1     (V <- V Q_{j-1})
// Every CTA asks for more than half an SM's shared memory, so each runs alone
// on its SM: the latency-bound solve CTAs do not share issue slots with the
// DMMA-bound update CTAs (sharing cost the solve ~5 us per round when the
// updates ran beside it as separate kernels), and for n <= 1024 the whole
// round fits in one wave of 148 CTAs. The round's duration is the solve's.
constexpr int AH_LX = 68, AH_LT = 36;
constexpr int FR_THREADS = 384;        // worker CTAs: 12 warps (3 per SM quadrant; 16 spill and ran slower)
constexpr int FR_SOLVE_THREADS = 256;  // solve CTAs: 8 warps form the subproblem, 4 of them run the rounds
constexpr size_t FR_SMEM_USED = (64 * AH_LX + 32 * AH_LT + 32 * AH_LX + 32 * AH_LT) * sizeof(double);
constexpr size_t FR_SMEM = 116 * 1024;  // > 227 KB / 2: one CTA per SM
static_assert(FR_SMEM >= FR_SMEM_USED, "fused-round shared memory");

template <bool FAST>
__device__ __forceinline__ void fused_solve_role(const double* A, int64_t lda, const SolveTables<32>* tabs,
                                                 double* Qbuf, int* active, int nb, int round,
                                                 const double* skip_tau_p, int mode, const double* Qprev,
                                                 const int* act_prev, int rprev, int pair) {
    constexpr int TB = 32, B = 16, QW = 4, QR = 8;
    extern __shared__ double dsm[];
    double* X = dsm;                 // 64 x 64, ld AH_LX
    double* Tc = X + 64 * AH_LX;     // 32 x 32, ld AH_LT: columns 0-15 = T_I, 16-31 = T_J
    double* Y = Tc + 32 * AH_LT;     // 64 x 32, ld AH_LX
    double* Ms = Y + 32 * AH_LX;     // 32 x 32, ld AH_LT
    __shared__ __align__(16) unsigned char sched[TB - 1][TB];
    __shared__ double pd[2][QW][TB], px[2][QW][TB];
    __shared__ int prev[4];  // p_I, offset of I in it, p_J, offset of J
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid >= FR_SOLVE_THREADS) return;  // the role's barriers count FR_SOLVE_THREADS threads
    const int r = lane >> 2, kq = lane & 3;
    const int R = mode == 0 ? TB - 1 : (mode == 1 ? B - 1 : B);
    const bool probe = pair == 0 && round == 5 && tid == 0;
    const long long t0 = SVDK_CLOCK();
#ifdef SVDK_PROBES
    const bool tl = pair == 0 && tid == 0 && round < 16 && mode == 2;
    if (tl) g_jtimeline[round * 8 + 0] = gtime();
#endif
    int I, J;
    circle_pair(nb, round, pair, I, J);
    {
        const uint4* src = reinterpret_cast<const uint4*>(&tabs[mode].part[0][0]);
        uint4* dst = reinterpret_cast<uint4*>(&sched[0][0]);
        for (int e = tid; e < static_cast<int>(sizeof(sched) / 16); e += FR_SOLVE_THREADS) dst[e] = src[e];
        if (rprev >= 0) {  // where I and J sat in the previous round (independent of its results)
            for (int i = tid; i < nb / 2; i += FR_SOLVE_THREADS) {
                int a, b;
                circle_pair(nb, rprev, i, a, b);
                if (a == I) { prev[0] = i; prev[1] = 0; }
                if (b == I) { prev[0] = i; prev[1] = B; }
                if (a == J) { prev[2] = i; prev[3] = 0; }
                if (b == J) { prev[2] = i; prev[3] = B; }
            }
        }
    }
    named_bar(2, FR_SOLVE_THREADS);
    pdl_wait();  // the previous kernel: Q_{j-1}, its active flags and A_{j-2}
    const long long t1 = SVDK_CLOCK();
#ifdef SVDK_PROBES
    if (tl) g_jtimeline[round * 8 + 1] = gtime();
#endif
    const double skip_tau = *skip_tau_p;
    const int row0 = (w & 3) * QR;
    double wreg[QR], qreg[QR];
    if (rprev < 0) {
        if (w < QW) {
            const double* col = A + gidx(B, I, J, row0) + gidx(B, I, J, lane) * lda;
#pragma unroll
            for (int v = 0; v < QR / 4; ++v) {
                const double4 x = ld_cg4(col + 4 * v);
                wreg[4 * v] = x.x; wreg[4 * v + 1] = x.y; wreg[4 * v + 2] = x.z; wreg[4 * v + 3] = x.w;
            }
        }
    } else {
        const int pI = prev[0], oI = prev[1], pJ = prev[2], oJ = prev[3];
        int bl[4];
        circle_pair(nb, rprev, pI, bl[0], bl[1]);
        circle_pair(nb, rprev, pJ, bl[2], bl[3]);
        // X = A_{j-2}[P, P]: 1024 four-row vectors, 4 per thread, all in flight; T: 256, 1 per thread
        double4 xv[4], tv;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int e = tid + FR_SOLVE_THREADS * k, c = e >> 4, r4 = (e & 15) * 4;
            xv[k] = ld_cg4(A + static_cast<int64_t>(bl[r4 >> 4]) * B + (r4 & 15) +
                           (static_cast<int64_t>(bl[c >> 4]) * B + (c & 15)) * lda);
        }
        {
            const int c = tid >> 3, r4 = (tid & 7) * 4;
            const int pp = c < B ? pI : pJ, cc = c < B ? oI + c : oJ + (c - B);
            // the slot is read unconditionally (always allocated), beside the flag instead of behind it
            const int act = __ldcg(&act_prev[pp]);
            tv = ld_cg4(Qprev + static_cast<size_t>(pp) * 1024 + r4 + cc * 32);
            if (!act) tv = make_double4(r4 == cc, r4 + 1 == cc, r4 + 2 == cc, r4 + 3 == cc);
            double* d = Tc + r4 + c * AH_LT;
            d[0] = tv.x; d[1] = tv.y; d[2] = tv.z; d[3] = tv.w;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int e = tid + FR_SOLVE_THREADS * k, c = e >> 4, r4 = (e & 15) * 4;
            double* d = X + r4 + c * AH_LX;
            d[0] = xv[k].x; d[1] = xv[k].y; d[2] = xv[k].z; d[3] = xv[k].w;
        }
        named_bar(2, FR_SOLVE_THREADS);
        {  // Y = X T: warp w forms rows [8w, 8w + 8); n-tiles 0, 1 contract over P's first pair, 2, 3 over its
           // second. M's lower-left block is the mirror of its upper-right one, so rows 32.. of Y (warps 4-7)
           // only need the n-tiles 2, 3.
            const int t0 = w < 4 ? 0 : 2;
            double acc[4][2];
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
            for (int s8 = 0; s8 < 8; ++s8) {
                const int k = 4 * s8 + kq;
                const double a1 = X[(8 * w + r) + (32 + k) * AH_LX];
                if (t0 == 0) {
                    const double a0 = X[(8 * w + r) + k * AH_LX];
#pragma unroll
                    for (int t = 0; t < 2; ++t) dmma(acc[t][0], acc[t][1], a0, Tc[k + (8 * t + r) * AH_LT]);
                }
#pragma unroll
                for (int t = 2; t < 4; ++t) dmma(acc[t][0], acc[t][1], a1, Tc[k + (8 * t + r) * AH_LT]);
            }
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    if (t >= t0) Y[(8 * w + r) + (8 * t + 2 * kq + i) * AH_LX] = acc[t][i];
        }
        named_bar(2, FR_SOLVE_THREADS);
        {  // M = T^T Y: warp w forms rows [8 (w & 3), + 8) x columns [16 (w >> 2), + 16); the lower-left block
           // (rows >= 16, columns < 16) is read as the mirror of the upper-right one below
            const int mw = w & 3, nh = w >> 2;
            if (!(mw >= 2 && nh == 0)) {
                double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
                const int yoff = mw < 2 ? 0 : 32;  // rows < 16: T_I^T Y[0:32], else T_J^T Y[32:64]
#pragma unroll
                for (int s8 = 0; s8 < 8; ++s8) {
                    const int k = 4 * s8 + kq;
                    const double af = Tc[k + (8 * mw + r) * AH_LT];
#pragma unroll
                    for (int t = 0; t < 2; ++t)
                        dmma(acc[t][0], acc[t][1], af, Y[(yoff + k) + (8 * (2 * nh + t) + r) * AH_LX]);
                }
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int i = 0; i < 2; ++i)
                        Ms[(8 * mw + r) + (8 * (2 * nh + t) + 2 * kq + i) * AH_LT] = acc[t][i];
            }
        }
        named_bar(2, FR_SOLVE_THREADS);
        if (w < QW) {
#pragma unroll
            for (int i = 0; i < QR; ++i) {
                const int rw = row0 + i;
                wreg[i] = (rw >= 16 && lane < 16) ? Ms[lane + rw * AH_LT] : Ms[rw + lane * AH_LT];
            }
        }
    }
    bool big = false;
    if (w < QW) {
#pragma unroll
        for (int i = 0; i < QR; ++i) {
            big |= (row0 + i != lane) && fabs(wreg[i]) > skip_tau;
            qreg[i] = (row0 + i == lane) ? 1.0 : 0.0;
        }
    }
    const bool work = named_bar_or(2, FR_SOLVE_THREADS, big);
    if (tid == 0) active[pair] = work ? 1 : 0;
    if (w >= QW || !work) return;  // warps 4-7 only helped with the subproblem
    if (probe) {
        SVDK_PROBE_STORE(g_jprobe, 0, t0);
        SVDK_PROBE_STORE(g_jprobe, 1, t1);
        SVDK_PROBE_STORE(g_jprobe, 2, SVDK_CLOCK());
    }
    os_rounds<QR, QW, FAST>(qreg, wreg, sched, R, R, pd, px, w, lane, 1, skip_tau);
    if (probe) SVDK_PROBE_STORE(g_jprobe, 3, SVDK_CLOCK());
    // column-norm Newton step (see jacobi_pair_solve_os)
    double n0 = qreg[0] * qreg[0], n1 = qreg[1] * qreg[1];
#pragma unroll
    for (int i = 2; i < QR; i += 2) {
        n0 = fma(qreg[i], qreg[i], n0);
        n1 = fma(qreg[i + 1], qreg[i + 1], n1);
    }
    const int buf = R & 1;
    pd[buf][w][lane] = n0 + n1;
    named_bar(1, 32 * QW);
    const double nn = (pd[buf][0][lane] + pd[buf][1][lane]) + (pd[buf][2][lane] + pd[buf][3][lane]);
    const double f = fma(-0.5, nn, 1.5);
    double* out = Qbuf + static_cast<size_t>(pair) * TB * TB + row0 + lane * TB;
#pragma unroll
    for (int v = 0; v < QR / 4; ++v)
        st4(out + 4 * v, f * qreg[4 * v], f * qreg[4 * v + 1], f * qreg[4 * v + 2], f * qreg[4 * v + 3]);
    if (probe) SVDK_PROBE_STORE(g_jprobe, 4, SVDK_CLOCK());
#ifdef SVDK_PROBES
    if (tl) g_jtimeline[round * 8 + 2] = gtime();
#endif
}

template <bool FAST>
__global__ void __launch_bounds__(FR_THREADS, 1)
    jacobi_round_fused(const double* Ain, double* Aout, double* V, int64_t ld, const SolveTables<32>* tabs,
                       double* Qcur, int* act_cur, const double* Qprev, const int* act_prev, int nb, int round,
                       int rprev, int mode, const double* skip_tau_p, int n_solve, int a_tasks, int v_tasks) {
    const int b = blockIdx.x, w = threadIdx.x >> 5;
    // Every CTA lets the next round's kernel launch at once: its CTAs take the SMs this kernel leaves
    // free (one CTA per SM, so they crowd nobody), run their prologue up to griddepcontrol.wait and
    // absorb the launch latency (n = 256: 0.8 us gap + 0.5 us prologue per round, tools/fr_timeline.py).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (b < n_solve) {
        fused_solve_role<FAST>(Ain, ld, tabs, Qcur, act_cur, nb, round, skip_tau_p, mode, Qprev, act_prev, rprev, b);
        return;
    }
    // worker CTAs: warp tasks of round j-1's updates, grid-strided. A task: one
    // half (16 rows) of a 32 x 32 unit of A_{j-1} = Q^T A_{j-2} Q; V task: one
    // (pair, 32-row chunk) of V <- V Q.
    const bool probe = b == n_solve && threadIdx.x == 0 && round == 5;
    const long long t0 = SVDK_CLOCK();
#ifdef SVDK_PROBES
    const bool tl = threadIdx.x == 0 && round < 16 && mode == 2 && n_solve > 0;
    if (tl && b == n_solve) g_jtimeline[round * 8 + 3] = gtime();
#endif
    pdl_wait();
#ifdef SVDK_PROBES
    if (tl && b == n_solve) g_jtimeline[round * 8 + 4] = gtime();
#endif
    if (probe) {
        SVDK_PROBE_STORE(g_jprobe, 8, t0);
        SVDK_PROBE_STORE(g_jprobe, 9, SVDK_CLOCK());
    }
    const int nw = (gridDim.x - n_solve) * (FR_THREADS / 32);
    for (int t = (b - n_solve) * (FR_THREADS / 32) + w; t < a_tasks + v_tasks; t += nw) {
        if (t < a_tasks)
            upd_a_unit_vec<2, false>(Ain, Aout, ld, Qprev, act_prev, nb, rprev, t >> 1, t & 1);
        else
            upd_v_unit(V, ld, ld, Qprev, act_prev, nb, rprev, t - a_tasks, 32);
        if (probe && t < nw) SVDK_PROBE_STORE(g_jprobe, 10, SVDK_CLOCK());
    }
    if (probe) SVDK_PROBE_STORE(g_jprobe, 11, SVDK_CLOCK());
#ifdef SVDK_PROBES
    if (tl && b == n_solve) g_jtimeline[round * 8 + 5] = gtime();
    if (tl) atomicMax(&g_jtimeline[round * 8 + 6], gtime());
#endif
}

// ---------------------------------------------------------------------------
// setup / checks / finish
// ---------------------------------------------------------------------------
// max|s_ij| and max|s_ij - s_ji| (block partials; max is order-independent)
__global__ void symcheck_kernel(const double* S, int64_t lds, int64_t n, double* partial) {
    __shared__ double r1[32], r2[32];
    double mabs = 0.0, masym = 0.0;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / n, i = e - j * n;
        const double a = S[i + j * lds];
        mabs = fmax(mabs, fabs(a));
        masym = fmax(masym, fabs(a - S[j + i * lds]));
    }
    for (int o = 16; o > 0; o >>= 1) {
        mabs = fmax(mabs, __shfl_xor_sync(0xffffffffu, mabs, o));
        masym = fmax(masym, __shfl_xor_sync(0xffffffffu, masym, o));
    }
    if ((threadIdx.x & 31) == 0) {
        r1[threadIdx.x >> 5] = mabs;
        r2[threadIdx.x >> 5] = masym;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (blockDim.x >> 5); ++w) {
            mabs = fmax(mabs, r1[w]);
            masym = fmax(masym, r2[w]);
        }
        partial[2 * blockIdx.x] = mabs;
        partial[2 * blockIdx.x + 1] = masym;
    }
}

// A (n_pad x n_pad) = (S + S^T)/2 zero padded; V = I.
__global__ void jacobi_init_kernel(const double* S, int64_t lds, int64_t n, double* A, double* V,
                                   int64_t n_pad, const double* scale_p) {
    const double scale = *scale_p;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n_pad * n_pad;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / n_pad, i = e - j * n_pad;
        double a = 0.0;
        if (i < n && j < n) a = (0.5 * (S[i + j * lds] + S[j + i * lds])) * scale;
        A[e] = a;
        V[e] = (i == j) ? 1.0 : 0.0;
    }
}

// partial sums of squares: mode 0 = all entries, mode 1 = strictly lower.
// Block b sums the columns b, b + grid, ... (rows i > j in mode 1), coalesced
// along the column, with a fixed order: deterministic partials.
__global__ void jacobi_sumsq_kernel(const double* A, int64_t n, int mode, double* partial) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
        const double* col = A + j * n;
        for (int64_t i = (mode ? j + 1 : 0) + threadIdx.x; i < n; i += blockDim.x) s = fma(col[i], col[i], s);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (blockDim.x >> 5); ++w) s += red[w];
        partial[blockIdx.x] = s;
    }
}

// Stable descending order by rank counting: rank_i = #{j : l_j > l_i or
// (l_j == l_i and j < i)} — exactly std::stable_sort's permutation.
__global__ void eig_sort_kernel(const double* A, int64_t n_pad, int64_t n, const double* unscale_p,
                                double* w, int* dest) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double unscale = *unscale_p;
    const double li = A[i + i * n_pad];
    int64_t rank = 0;
    for (int64_t j = 0; j < n; ++j) {
        const double lj = A[j + j * n_pad];
        rank += (lj > li) || (lj == li && j < i);
    }
    w[rank] = li * unscale;
    dest[i] = static_cast<int>(rank);
}

__global__ void eig_gather_kernel(const double* V, int64_t n_pad, int64_t n, const int* dest,
                                  double* Vout, int64_t ldv) {
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
        const int64_t d = dest[j];
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            Vout[i + d * ldv] = V[i + j * n_pad];
    }
}

// Convergence test of one sweep on the device: off = sqrt(2 sum partial)
// (fixed order, as device_sumsq), sweep counter, and the WHILE condition of
// the enclosing graph: keep sweeping while off > thr and sweeps < max_sweeps
// (kernels.cpp:274-326, the host loop's exact test).
// Device scalars of a sweep loop (JS_* slots of `scal`), written by
// jacobi_start_kernel / eig_prep_kernel and read by the sweep kernels, so the
// instantiated graphs never bake a per-call value.
enum { JS_THR = 0, JS_SKIP, JS_OFF, JS_SWEEPS, JS_SCALE, JS_UNSCALE, JS_MABS, JS_MASYM, JS_MAXSW, JS_FRO,
       JS_POLISH, JS_CONT, JS_POLISH_ON, JS_COUNT };

// Fixed-order warp sum / max of count partials (lane-strided sequential sums
// then a fixed xor tree: deterministic, ~30x shorter than one thread's loop).
__device__ __forceinline__ double warp_sum_fixed(const double* partial, int count) {
    double s = 0.0;
    for (int i = threadIdx.x; i < count; i += 32) s += partial[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// After a sweep: off(A) from the partials; continue while off > thr and
// sweeps < max_sweeps (kernels.cpp:274-326). Once converged, ONE polish sweep
// follows (JS_POLISH 0 -> 1 -> 2): the block-parallel order leaves its last
// sweep's small couplings between close eigenvalues (per-vector sines ~1e-8
// at c4's relative gaps ~1e-6, vs ~3e-9 for two independent exact solvers);
// the polish squares them away. off and the sweep count reported to the
// caller stay those of the converged sweep, so the error contract and the
// sweep trajectory are the reference's.
__global__ void jacobi_decide_kernel(cudaGraphConditionalHandle h, const double* partial, int count,
                                     double* scal, int use_cond) {
    if (blockIdx.x != 0) return;
    const double s = warp_sum_fixed(partial, count);  // all 32 lanes
    if (threadIdx.x != 0) return;
    double cont = 0.0;
    if (scal[JS_POLISH] != 0.0) {
        scal[JS_POLISH] = 2.0;  // the polish sweep ran
    } else {
        const double off = sqrt(2.0 * s);
        const double sw = scal[JS_SWEEPS] + 1.0;
        scal[JS_OFF] = off;
        scal[JS_SWEEPS] = sw;
        if (off > scal[JS_THR]) {
            cont = sw < scal[JS_MAXSW] ? 1.0 : 0.0;
        } else if (scal[JS_POLISH_ON] != 0.0) {
            scal[JS_POLISH] = 1.0;
            cont = 1.0;
        }
    }
    scal[JS_CONT] = cont;
    if (use_cond) cudaGraphSetConditional(h, cont != 0.0 ? 1u : 0u);
}

// Before the first sweep (kernels.cpp:271-274): ||A||_F from the all-entries
// partials, thr = 1e-12 ||A||_F, the solves' skip threshold, off(A) from the
// strictly-lower partials; sweep only if off > thr (and max_sweeps > 0).
__global__ void jacobi_start_kernel(cudaGraphConditionalHandle h, const double* p_all, const double* p_low,
                                    int count, double n_pad, double* scal, int use_cond) {
    if (blockIdx.x != 0) return;
    const double s0 = warp_sum_fixed(p_all, count), s1 = warp_sum_fixed(p_low, count);
    if (threadIdx.x != 0) return;
    const double fro = sqrt(s0), off = sqrt(2.0 * s1);
    scal[JS_FRO] = fro;
    scal[JS_THR] = 1e-12 * fro;
    scal[JS_SKIP] = 1e-13 * fro / n_pad;
    scal[JS_OFF] = off;
    scal[JS_SWEEPS] = 0.0;
    scal[JS_POLISH] = 0.0;
    const double cont = (off > scal[JS_THR] && scal[JS_MAXSW] > 0.0) ? 1.0 : 0.0;
    scal[JS_CONT] = cont;
    if (use_cond) cudaGraphSetConditional(h, cont != 0.0 ? 1u : 0u);
}

// max|s_ij|, max|s_ij - s_ji| from symcheck_kernel's partials, the exact
// power-of-two prescale (entries whose squares cannot over/underflow) and
// the sweep cap, all on the device (no host round trip before the sweeps).
__global__ void eig_prep_kernel(const double* partial, int count, int max_sweeps, int polish, double* scal) {
    if (blockIdx.x != 0) return;
    double mabs = 0.0, masym = 0.0;
    for (int b = threadIdx.x; b < count; b += 32) {
        mabs = fmax(mabs, partial[2 * b]);
        masym = fmax(masym, partial[2 * b + 1]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mabs = fmax(mabs, __shfl_xor_sync(0xffffffffu, mabs, o));
        masym = fmax(masym, __shfl_xor_sync(0xffffffffu, masym, o));
    }
    if (threadIdx.x != 0) return;
    int pow2 = 0;
    if (mabs > 0.0 && (mabs > 1e100 || mabs < 1e-100)) pow2 = ilogb(mabs);
    scal[JS_SCALE] = ldexp(1.0, -pow2);
    scal[JS_UNSCALE] = ldexp(1.0, pow2);
    scal[JS_MABS] = mabs;
    scal[JS_MASYM] = masym;
    scal[JS_MAXSW] = static_cast<double>(max_sweeps);
    scal[JS_POLISH_ON] = polish ? 1.0 : 0.0;
}

// A sweep plan: the padded work matrices, the per-round rotation slots, the
// schedule tables and ONE instantiated graph holding every sweep of an
// eig_sym call — a WHILE conditional node whose body is the captured sweep
// (both streams) + the off-diagonal sum of squares + jacobi_decide_kernel,
// preceded by jacobi_start_kernel (threshold and first convergence test,
// kernels.cpp:271-274). Every per-call value (thresholds, prescale, sweep cap)
// lives in device scalars, so the plan is built once per (context, n_pad,
// scheme) and replayed by later calls: no capture / instantiation and no host
// round trip inside eig_sym (one read of the final scalars at the end).
}  // namespace

struct JacobiPlan {
    int64_t n_pad = 0;
    int tb = 0;  // 16 / 32: pair scheme, 64: quad scheme
    DBuf A, V, qbuf, act, tabs, part_all, part_low, scal;
    DBuf A2;  // solve-ahead: the other half of the A ping-pong pair
    int blocks = 0;  // sum-of-squares partial blocks
    int launches_per_sweep = 0;
    std::function<void()> enqueue_sweep;  // one sweep on (stream, aux stream)
    cudaGraphExec_t exec = nullptr;       // nullptr: host-driven sweep loop
    JacobiPlan() = default;
    JacobiPlan(const JacobiPlan&) = delete;
    JacobiPlan& operator=(const JacobiPlan&) = delete;
    ~JacobiPlan() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

struct JacobiCache {
    std::vector<std::unique_ptr<JacobiPlan>> plans;  // most recently used last
};

namespace {
constexpr size_t kMaxPlans = 4;

// Contexts of one process may be driven by several host threads (the host-staged
// group runs one rank per thread, and every rank of a sketch method solves its own
// small eigenproblem). Building a plan (stream capture into a conditional-node
// graph + instantiation) and launching one are serialised across threads: with
// them concurrent, tests/test_gpu_sharded.py's sketch cases died with SIGSEGV
// inside svdk_dev_pca in ~8% of runs.
std::mutex& graph_mutex() {
    static std::mutex mu;
    return mu;
}

cudaGraphNode_t add_kernel_node(cudaGraph_t g, const cudaGraphNode_t* deps, size_t ndeps, const void* func,
                                dim3 grid, dim3 block, void** args) {
    cudaKernelNodeParams kp = {};
    kp.func = const_cast<void*>(func);
    kp.gridDim = grid;
    kp.blockDim = block;
    kp.sharedMemBytes = 0;
    kp.kernelParams = args;
    cudaGraphNode_t node = nullptr;
    if (cudaGraphAddKernelNode(&node, g, deps, ndeps, &kp) != cudaSuccess) return nullptr;
    return node;
}

// Build P.exec = [sumsq(all), sumsq(lower)] -> start -> WHILE{sweep, sumsq(lower), decide}.
// Leaves P.exec null where conditional nodes are unavailable or disabled.
void build_loop_graph(Ctx* c, JacobiPlan& P) {
    if (const char* e = std::getenv("SVDK_JACOBI_DEVLOOP"))
        if (std::string(e) == "0") return;
    cudaStream_t S = c->stream;
    if (!S) return;
    cudaGraph_t outer = nullptr;
    if (cudaGraphCreate(&outer, 0) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    cudaGraphConditionalHandle h;
    if (cudaGraphConditionalHandleCreate(&h, outer, 0, cudaGraphCondAssignDefault) != cudaSuccess) {
        cudaGetLastError();
        cudaGraphDestroy(outer);
        return;
    }
    double* A = P.A.p();
    int64_t n = P.n_pad;
    int mode0 = 0, mode1 = 1;
    double* pa = P.part_all.p();
    double* pl = P.part_low.p();
    double* scal = P.scal.p();
    int blocks = P.blocks;
    double npad_d = static_cast<double>(P.n_pad);
    void* a0[] = {&A, &n, &mode0, &pa};
    void* a1[] = {&A, &n, &mode1, &pl};
    const cudaGraphNode_t s0 = add_kernel_node(outer, nullptr, 0, reinterpret_cast<const void*>(jacobi_sumsq_kernel),
                                               dim3(blocks), dim3(256), a0);
    const cudaGraphNode_t s1 = add_kernel_node(outer, nullptr, 0, reinterpret_cast<const void*>(jacobi_sumsq_kernel),
                                               dim3(blocks), dim3(256), a1);
    int use_cond = 1;
    void* as[] = {&h, &pa, &pl, &blocks, &npad_d, &scal, &use_cond};
    cudaGraphNode_t deps[2] = {s0, s1};
    const cudaGraphNode_t st = (s0 && s1) ? add_kernel_node(outer, deps, 2, reinterpret_cast<const void*>(
                                                                jacobi_start_kernel), dim3(1), dim3(32), as)
                                          : nullptr;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    if (!st || cudaGraphAddNode(&cnode, outer, &st, 1, &cp) != cudaSuccess) {
        cudaGetLastError();
        cudaGraphDestroy(outer);
        return;
    }
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if (cudaStreamBeginCaptureToGraph(S, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
        cudaSuccess) {
        cudaGetLastError();
        cudaGraphDestroy(outer);
        return;
    }
    // A capture can be invalidated from outside (e.g. another host thread calls
    // cudaDeviceSynchronize while this stream captures): any failure here leaves
    // P.exec null and eig_sym drives the same kernels from the host instead.
    cudaGraph_t captured = nullptr;
    bool captured_ok = true;
    try {
        P.enqueue_sweep();
        jacobi_sumsq_kernel<<<blocks, 256, 0, S>>>(A, n, 1, pl);
        jacobi_decide_kernel<<<1, 32, 0, S>>>(h, pl, blocks, scal, 1);
    } catch (const Failure&) {
        captured_ok = false;
    } catch (...) {  // leave the stream out of capture mode
        cudaStreamEndCapture(S, &captured);
        cudaGetLastError();
        cudaGraphDestroy(outer);
        throw;
    }
    if (cudaStreamEndCapture(S, &captured) != cudaSuccess || !captured_ok) {
        cudaGetLastError();
        cudaGraphDestroy(outer);
        return;
    }
    const cudaError_t ie = cudaGraphInstantiate(&P.exec, outer, 0);
    cudaGraphDestroy(outer);
    if (ie != cudaSuccess) {
        cudaGetLastError();
        P.exec = nullptr;
    }
}

// Run the plan's sweeps on the work matrices (already initialised): the
// graph when there is one, else the same kernels driven from the host.
// Returns the sweep count; scal holds off / thr.
int run_plan(Ctx* c, JacobiPlan& P) {
    cudaStream_t S = c->stream;
    if (P.exec) {
        std::lock_guard<std::mutex> lock(graph_mutex());
        SVDK_CUDA(cudaGraphLaunch(P.exec, S));
        return -1;  // read from scal by the caller
    }
    double* scal = P.scal.p();
    cudaGraphConditionalHandle none{};
    jacobi_sumsq_kernel<<<P.blocks, 256, 0, S>>>(P.A.p(), P.n_pad, 0, P.part_all.p());
    jacobi_sumsq_kernel<<<P.blocks, 256, 0, S>>>(P.A.p(), P.n_pad, 1, P.part_low.p());
    jacobi_start_kernel<<<1, 32, 0, S>>>(none, P.part_all.p(), P.part_low.p(), P.blocks,
                                         static_cast<double>(P.n_pad), scal, 0);
    SVDK_CHECK_LAUNCH();
    c->launches += 3;
    double h[JS_COUNT];
    d2h(c, h, scal, JS_COUNT);
    while (h[JS_CONT] != 0.0) {
        P.enqueue_sweep();
        SVDK_CHECK_LAUNCH();
        jacobi_sumsq_kernel<<<P.blocks, 256, 0, S>>>(P.A.p(), P.n_pad, 1, P.part_low.p());
        jacobi_decide_kernel<<<1, 32, 0, S>>>(none, P.part_low.p(), P.blocks, scal, 0);
        SVDK_CHECK_LAUNCH();
        c->launches += P.launches_per_sweep + 2;
        d2h(c, h, scal, JS_COUNT);
    }
    return static_cast<int>(h[JS_SWEEPS]);
}

// Largest n_pad that runs the solve-ahead chain by default (see jacobi_pair_solve_ahead).
// Measured (eig_sym ms, fused / separate kernels): n = 1024 8.9 / 10.8, 1152 10.3 / 13.4, 1280 16.1 / 15.5,
// 1536 25.9 / 25.2, 1792 42.2 / 32.9, 2048 86.6 / 45.2 — above ~1200 the worker CTAs' task throughput
// (one CTA per SM) falls behind the separate update kernels.
constexpr int64_t kAheadMaxN = 1152;

template <int TB>
void build_pair_plan(Ctx* c, JacobiPlan& P) {
    constexpr int B = TB / 2;
    const int64_t n_pad = P.n_pad;
    const int nb = static_cast<int>(n_pad / B);
    const int k = nb / 2;
    const size_t smem_solve = 4 * TB * (TB + 4) * sizeof(double);
    constexpr int nthreads_solve = solve_threads<TB>();
    const size_t smem_a = 4 * TB * (TB + 4) * sizeof(double);
    const size_t smem_v = 3 * TB * (TB + 4) * sizeof(double);
    ensure_smem_attr(reinterpret_cast<const void*>(jacobi_pair_solve<TB>), smem_solve);
    ensure_smem_attr(reinterpret_cast<const void*>(jacobi_update_a<TB>), smem_a);
    ensure_smem_attr(reinterpret_cast<const void*>(jacobi_update_v<TB>), smem_v);
    // Inner skip threshold (JS_SKIP): if every off-diagonal entry were this
    // small the outer test off <= 1e-12 ||A||_F would hold with a 10x margin.
    const char* inner_env = std::getenv("SVDK_JACOBI_INNER");
    const int max_inner = inner_env ? std::max(1, std::atoi(inner_env)) : 1;
    const int rounds = nb - 1;
    // Schedule: "split" (default) rotates every index pair exactly once per
    // sweep, like the reference's cyclic sweep: a first stage diagonalises
    // pairs inside each b-block (mode 1), then the nb-1 tournament rounds
    // rotate only the cross pairs of each block pair (mode 2, b inner rounds
    // instead of 2b-1). "full" (SVDK_JACOBI_SCHEME=full) re-rotates the
    // in-block pairs in every round (mode 0).
    const char* scheme_env = std::getenv("SVDK_JACOBI_SCHEME");
    const bool split = !(scheme_env && std::string(scheme_env) == "full");
    const int slots = rounds + (split ? 1 : 0);
    // Every round of a sweep keeps its own Q_p set, so the V chain on the side
    // stream can lag behind the A chain by any number of rounds.
    P.qbuf = DBuf(c, static_cast<size_t>(slots) * k * TB * TB);
    P.act = DBuf(c, static_cast<size_t>(slots) * k);
    int* active = reinterpret_cast<int*>(P.act.p());
    const int a_ctas = k * (k + 1) / 2, v_ctas = static_cast<int>(n_pad / TB) * k;
    if (!c->aux_stream) {
        SVDK_CUDA(cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
        SVDK_CUDA(cudaEventCreateWithFlags(&c->aux_ev[0], cudaEventDisableTiming));
        SVDK_CUDA(cudaEventCreateWithFlags(&c->aux_ev[1], cudaEventDisableTiming));
    }
    cudaStream_t S = c->stream;
    // register-resident updates for 2b = 32 (SVDK_JACOBI_UPD=smem: the
    // shared-memory kernels, kept for TB = 16 and for comparison)
    const char* upd_env = std::getenv("SVDK_JACOBI_UPD");
    const bool reg_upd = TB == 32 && !(upd_env && std::string(upd_env) == "smem");
    const int a_warp_ctas = static_cast<int>(ceil_div(static_cast<int64_t>(a_ctas), UPD_WARPS));
    // Default: the vector-load, shuffle-free unit (upd_a_unit_vec) with 2 warps
    // per unit up to n = 1024 and 1 above. Measured eig(n) in ms, same box
    // (tools/exp_probe.py; SVDK_JACOBI_AVEC = warps per unit, 0 = upd_a_unit,
    // SVDK_JACOBI_AQ4=1 = jacobi_update_a_q4):
    //   n        256   512   1024  2048  3000
    //   vec x1  3.39  6.97  16.70  54.3   161
    //   vec x2  3.23  6.28  15.52  59.7   182
    //   vec x4  3.27  6.40  15.79  56.7   175
    //   q4      3.23  6.57  17.23
    //   reg          (1024: 16.62, 2048: 58.6, 3000: 167.7 in another run)
    const char* q4_env = std::getenv("SVDK_JACOBI_AQ4");
    const bool a_q4 = q4_env && std::atoi(q4_env) != 0;
    const char* avec_env = std::getenv("SVDK_JACOBI_AVEC");
    const int a_vec = avec_env ? std::atoi(avec_env) : (n_pad <= 1024 ? 2 : 1);
    const int a_ctas2 = static_cast<int>(ceil_div(static_cast<int64_t>(a_ctas), 2));
    const int v_warp_ctas =
        static_cast<int>(ceil_div(ceil_div(n_pad, static_cast<int64_t>(VT_ROWS)) * k, UPD_WARPS));
    // Programmatic dependent launches on the solve -> A update -> solve chain
    // (SVDK_JACOBI_PDL=0: plain launches; see pdl_wait for the measurements).
    // Every kernel waits (griddepcontrol.wait) before reading its
    // predecessor's output; the solve's schedule tables come from the plan's
    // tables kernel, which completed before any sweep was enqueued.
    const char* pdl_env = std::getenv("SVDK_JACOBI_PDL");
    const bool pdl = !(pdl_env && std::atoi(pdl_env) == 0);
    // Pair solve: the one-sided kernel with SVDK_JACOBI_OS warps (2 / 4 / 8; 0 =
    // the two-sided solve_pair with its M threads and lookahead warp).
    const char* os_env = std::getenv("SVDK_JACOBI_OS");
    const int os_warps = os_env ? std::atoi(os_env) : 4;
    // SVDK_JACOBI_NS=1: Newton-Schulz on the accumulated rotation instead of the column-norm step
    const char* ns_env = std::getenv("SVDK_JACOBI_NS");
    const bool os_ns = ns_env && std::atoi(ns_env) != 0;
    const char* fast_env = std::getenv("SVDK_JACOBI_FASTROT");
    const bool os_fast = !(fast_env && std::atoi(fast_env) == 0);
    // timing-only development switches (results are wrong): bit 0 drops the A
    // update from the chain, bit 1 the V update
    const char* dbg_env = std::getenv("SVDK_JACOBI_DBG");
    const int dbg = dbg_env ? std::atoi(dbg_env) : 0;
    P.tabs = DBuf(c, 3 * sizeof(SolveTables<TB>) / sizeof(double));
    jacobi_tables_kernel<TB><<<3, 256, 0, S>>>(reinterpret_cast<SolveTables<TB>*>(P.tabs.p()));
    SVDK_CHECK_LAUNCH();
    c->launches++;
    const auto* tabs = reinterpret_cast<const SolveTables<TB>*>(P.tabs.p());
    double* A = P.A.p();
    double* V = P.V.p();
    const double* skip_p = P.scal.p() + JS_SKIP;
    double* qbase = P.qbuf.p();
    P.launches_per_sweep = 3 * slots;
    P.enqueue_sweep = [=]() {
        // the context's streams at enqueue time (svdk_ctx_set_stream may have moved them)
        const cudaStream_t S = c->stream, S2 = c->aux_stream;
        const cudaEvent_t ev0 = c->aux_ev[0], ev1 = c->aux_ev[1];
        auto launch = [&](auto kern, int grid, int block, size_t smem, bool prog, auto... args) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(static_cast<unsigned>(grid));
            cfg.blockDim = dim3(static_cast<unsigned>(block));
            cfg.dynamicSmemBytes = smem;
            cfg.stream = S;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = (prog && pdl) ? 1 : 0;
            SVDK_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
        };
        auto launch_updates = [&](const double* qr, const int* ar, int r) {
            if (reg_upd) {
                if (!(dbg & 2))
                    jacobi_update_v_reg<<<v_warp_ctas, UPD_WARPS * 32, 0, S2>>>(V, n_pad, n_pad, qr, ar, nb, r);
                int64_t ld = n_pad;
                const double* ac = A;
                if (dbg & 1) return;
                if (a_q4)
                    launch(jacobi_update_a_q4, a_ctas, 128, 0, true, A, ld, qr, ar, nb, r);
                else if (a_vec == 1)
                    launch(jacobi_update_a_vec<1>, a_warp_ctas, UPD_WARPS * 32, 0, true, ac, A, ld, qr, ar, nb, r);
                else if (a_vec == 2)
                    launch(jacobi_update_a_vec<2>, a_ctas2, UPD_WARPS * 32, 0, true, ac, A, ld, qr, ar, nb, r);
                else if (a_vec == 4)
                    launch(jacobi_update_a_vec<4>, a_ctas, UPD_WARPS * 32, 0, true, ac, A, ld, qr, ar, nb, r);
                else
                    launch(jacobi_update_a_reg, a_warp_ctas, UPD_WARPS * 32, 0, true, A, ld, qr, ar, nb, r);
            } else {
                jacobi_update_v<TB><<<v_ctas, 256, smem_v, S2>>>(V, n_pad, qr, ar, nb, r);
                jacobi_update_a<TB><<<a_ctas, 256, smem_a, S>>>(A, n_pad, qr, ar, nb, r);
            }
        };
        auto launch_solve = [&](double* qr, int* ar, int r, int mode) {
            const double* a = A;
            int64_t ld = n_pad;
            if constexpr (TB == 32) {
                auto go = [&](auto kern, int threads) {
                    launch(kern, k, threads, 0, true, a, ld, tabs, qr, ar, nb, r, skip_p, max_inner, mode);
                };
                if (os_warps == 8) {
                    go(os_ns ? (os_fast ? jacobi_pair_solve_os<8, true, true> : jacobi_pair_solve_os<8, true, false>)
                             : (os_fast ? jacobi_pair_solve_os<8, false, true> : jacobi_pair_solve_os<8, false, false>),
                       256);
                    return;
                }
                if (os_warps == 4) {
                    go(os_ns ? (os_fast ? jacobi_pair_solve_os<4, true, true> : jacobi_pair_solve_os<4, true, false>)
                             : (os_fast ? jacobi_pair_solve_os<4, false, true> : jacobi_pair_solve_os<4, false, false>),
                       128);
                    return;
                }
            }
            launch(jacobi_pair_solve<TB>, k, nthreads_solve, smem_solve, true, a, ld, tabs, qr, ar, nb, r, skip_p,
                   max_inner, mode);
        };
        if (split) {  // in-block stage on the round-0 block pairing
            double* qr = qbase + static_cast<size_t>(rounds) * k * TB * TB;
            int* ar = active + static_cast<size_t>(rounds) * k;
            launch_solve(qr, ar, 0, 1);
            SVDK_CUDA(cudaEventRecord(ev0, S));
            SVDK_CUDA(cudaStreamWaitEvent(S2, ev0, 0));
            launch_updates(qr, ar, 0);
        }
        for (int r = 0; r < rounds; ++r) {
            double* qr = qbase + static_cast<size_t>(r) * k * TB * TB;
            int* ar = active + static_cast<size_t>(r) * k;
            launch_solve(qr, ar, r, split ? 2 : 0);
            SVDK_CUDA(cudaEventRecord(ev0, S));
            SVDK_CUDA(cudaStreamWaitEvent(S2, ev0, 0));
            launch_updates(qr, ar, r);
        }
        // join: the sweep ends when the V chain has caught up
        SVDK_CUDA(cudaEventRecord(ev1, S2));
        SVDK_CUDA(cudaStreamWaitEvent(S, ev1, 0));
    };
    // Fused round kernels (jacobi_round_fused, solve-ahead): default for
    // n_pad <= kAheadMaxN, where a round is a latency chain; SVDK_JACOBI_AHEAD=0/1 overrides.
    bool ahead = TB == 32 && split && nb > 2 && n_pad <= kAheadMaxN && os_warps == 4 && !os_ns;
    if (const char* e = std::getenv("SVDK_JACOBI_AHEAD")) ahead = TB == 32 && split && nb > 2 && std::atoi(e) != 0;
    if constexpr (TB == 32) {
        if (ahead) {
            ensure_smem_attr(reinterpret_cast<const void*>(jacobi_round_fused<true>), FR_SMEM);
            ensure_smem_attr(reinterpret_cast<const void*>(jacobi_round_fused<false>), FR_SMEM);
            P.A2 = DBuf(c, static_cast<size_t>(n_pad) * n_pad);
            double* A2 = P.A2.p();
            const int a_tasks = 2 * a_ctas;  // half units
            const int v_tasks = static_cast<int>(n_pad / 32) * k;
            // worker CTAs: the SMs the solve CTAs leave free (every CTA runs alone on its SM), at
            // least `wtasks` warp tasks each (a task is DMMA-bound on its SM quadrant: one per quadrant)
            const char* wt_env = std::getenv("SVDK_JACOBI_FRTASKS");
            const int wtasks = wt_env ? std::max(1, std::atoi(wt_env)) : 4;
            int n_workers = static_cast<int>(std::max<int64_t>(
                1, std::min<int64_t>(c->num_sms - k, ceil_div(static_cast<int64_t>(a_tasks + v_tasks), wtasks))));
            if (const char* e = std::getenv("SVDK_JACOBI_FRWORKERS")) n_workers = std::max(1, std::atoi(e));  // tuning
            P.launches_per_sweep = slots + 1;
            const char* frs = std::getenv("SVDK_JACOBI_FRSMEM");  // KB, tuning: below 114 the roles share SMs
            const size_t fr_smem = frs ? std::max<size_t>(FR_SMEM_USED, static_cast<size_t>(std::atoi(frs)) * 1024) : FR_SMEM;
            P.enqueue_sweep = [=]() {
                const cudaStream_t S = c->stream;
                double* bufs[2] = {A, A2};
                const double* qprev = nullptr;
                const int* aprev = nullptr;
                int rprev = -1;
                int64_t ld = n_pad;
                // kernel j = {solve j, A and V updates j-1}; slots is even, so A is current at the end
                for (int j = 0; j <= slots; ++j) {
                    const bool has_solve = j < slots;
                    const int r = j == 0 ? 0 : j - 1, mode = j == 0 ? 1 : 2;
                    const size_t slot = j == 0 ? static_cast<size_t>(rounds) : static_cast<size_t>(r);
                    double* qr = qbase + slot * k * TB * TB;
                    int* ar = active + slot * k;
                    const int ns = (has_solve && !(dbg & 4)) ? k : 0, na = (j && !(dbg & 1)) ? a_tasks : 0,
                              nv = (j && !(dbg & 2)) ? v_tasks : 0, nwk = (na + nv) ? n_workers : 0;
                    if (ns + nwk == 0) {
                        qprev = qr;
                        aprev = ar;
                        rprev = r;
                        continue;
                    }
                    const double* a_in = j == 0 ? bufs[0] : bufs[(j - 1) & 1];
                    double* a_out = bufs[j & 1];
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(static_cast<unsigned>(ns + nwk));
                    cfg.blockDim = dim3(FR_THREADS);
                    cfg.dynamicSmemBytes = fr_smem;
                    cfg.stream = S;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    at[0].val.programmaticStreamSerializationAllowed = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = pdl ? 1 : 0;
                    if (os_fast)
                        SVDK_CUDA(cudaLaunchKernelEx(&cfg, jacobi_round_fused<true>, a_in, a_out, V, ld, tabs, qr, ar, qprev,
                                                     aprev, nb, r, rprev, mode, skip_p, ns, na, nv));
                    else
                        SVDK_CUDA(cudaLaunchKernelEx(&cfg, jacobi_round_fused<false>, a_in, a_out, V, ld, tabs, qr, ar,
                                                     qprev, aprev, nb, r, rprev, mode, skip_p, ns, na, nv));
                    qprev = qr;
                    aprev = ar;
                    rprev = r;
                }
            };
        }
    }
    if (nb > 2) build_loop_graph(c, P);
}

// ---------------------------------------------------------------------------
// 3. quad scheme: 64-wide updates (two 16-block rounds per similarity)
// ---------------------------------------------------------------------------
// The indices are cut into blocks of 16 and SUPER-blocks of 32 (blocks 2s,
// 2s+1). A sweep is the ns-1 rounds of a round-robin tournament over the ns
// super-blocks; in round r, super-pair (S, T) = ({I, J}, {K, L}) owns the
// 64 x 64 subproblem A[S T, S T] and rotates, as two 16-block "sub-stages"
// of two disjoint 32 x 32 cross solves each,
//     sub-stage B: (I, K) and (J, L)        sub-stage C: (I, L) and (J, K),
// i.e. all S x T cross pairs. Round 0 first runs sub-stage A: (I, J) and
// (K, L) with all pairs (mode 0), which covers every pair inside each super-
// block. So a sweep still rotates every index pair exactly once, like the
// reference's cyclic sweep, with the same 32 x 32 solve (and rotation
// formulas) as the 2b = 32 scheme; what changes is that the two sub-stages'
// rotations are composed into ONE 64 x 64 Q per super-pair inside the solve
// CTA (the second sub-stage sees the first one's similarity, applied to the
// 64 x 64 block in shared memory), so the full-matrix A and V updates run
// once per two 16-block rounds: half the HBM traffic for the same DMMA work
// (arithmetic intensity 8 instead of 4 flop/B, above the B200 FP64 ridge).
constexpr int L64 = 68;  // ld of 64 x 64 shared tiles (== 4 mod 16: conflict-free fragment loads)
constexpr int L32 = 36;
constexpr int QH = 256 + 128 + 32;  // threads per 32 x 32 solve: M threads, 4 Q warps, lookahead warp
constexpr int Q_THREADS = 2 * QH;  // two concurrent solves per CTA
constexpr int SUB32 = 32 * L32;
static_assert(QH == solve_threads<32>(), "solve roles");
constexpr size_t QUAD_SMEM =
    (3 * 64 * L64 + 8 * SUB32 + 4 * 31 * 16) * sizeof(double) + sizeof(SolveTables<32>) + 16;

// Local-64 index (blocks I J K L = 16-index groups 0..3) of local index i of
// half h's 32 x 32 subproblem in sub-stage `kind` (0 = A, 1 = B, 2 = C).
__device__ __forceinline__ int quad_idx(int kind, int h, int i) {
    if (kind == 0) return 32 * h + i;                    // {I, J} | {K, L}
    if (kind == 1) return (i < 16 ? i : i + 16) + 16 * h;  // {I, K} | {J, L}
    return h ? 16 + i : (i < 16 ? i : i + 32);           // {I, L} | {J, K}
}

// One 32 x 32 solve of a quad sub-stage, run by the QH threads of one half
// (ltid in [0, QH)) and synchronised by named barrier `bar`: the inner rounds
// of solve_pair (same roles, same operation order), then the Newton-Schulz
// step. Mc holds the subproblem on entry; Ts holds the rotation on exit
// (identity when !work).
__device__ __forceinline__ void quad_sub_solve(double* Mc, double* Mn, double* Qs, double* Ts,
                                               const SolveTables<32>& st, double (*cs)[16],
                                               double (*sn)[16], int R, int ltid, int bar, bool work,
                                               double skip_tau) {
    constexpr int TB = 32, LD = L32, NP = 16, MT = 256, QR = 8, QT = 128;
    if (!work) {
        for (int e = ltid; e < TB * TB; e += QH) Ts[(e & 31) + (e >> 5) * LD] = (e & 31) == (e >> 5) ? 1.0 : 0.0;
        named_bar(bar, QH);
        return;
    }
    const auto& ptab = st.ptab;
    const auto& pinv = st.pinv;
    const int lane = ltid - (MT + QT);
    if (lane >= 0 && lane < NP) {
        const int code = ptab[0][lane];
        const int p = code & 255, q = code >> 8;
        const double x = Mc[p + q * LD];
        double c = 1.0, s = 0.0;
        if (fabs(x) > skip_tau) rotation(Mc[p + p * LD], Mc[q + q * LD], x, c, s);
        cs[0][lane] = c;
        sn[0][lane] = s;
    }
    double qreg[QR];
    const int qrow0 = ((ltid - MT) >> 5) * QR;
#pragma unroll
    for (int i = 0; i < QR; ++i) qreg[i] = (qrow0 + i == ((ltid - MT) & 31)) ? 1.0 : 0.0;
    named_bar(bar, QH);
    for (int rr = 0; rr < R; ++rr) {
        if (ltid < MT + QT) {
            if (ltid < MT) {
                const int bi = ltid % NP, bj = ltid / NP;
                const int ci_code = ptab[rr][bi], cj_code = ptab[rr][bj];
                const int pi = ci_code & 255, qi = ci_code >> 8;
                const int pj = cj_code & 255, qj = cj_code >> 8;
                double m00 = Mc[pi + pj * LD], m01 = Mc[pi + qj * LD];
                double m10 = Mc[qi + pj * LD], m11 = Mc[qi + qj * LD];
                xform2x2(m00, m01, m10, m11, cs[rr][bi], sn[rr][bi], cs[rr][bj], sn[rr][bj], bi == bj);
                Mn[pi + pj * LD] = m00;
                Mn[pi + qj * LD] = m01;
                Mn[qi + pj * LD] = m10;
                Mn[qi + qj * LD] = m11;
            } else {
                const int l = (ltid - MT) & 31;
                const int code = pinv[rr][l];
                const int j = code & 127, role = code >> 7;
                const int pq = ptab[rr][j];
                const int partner = role ? (pq & 255) : (pq >> 8);
                const double c = cs[rr][j], b = role ? sn[rr][j] : -sn[rr][j];
#pragma unroll
                for (int i = 0; i < QR; ++i) {
                    const double other = __shfl_sync(0xffffffffu, qreg[i], partner);
                    qreg[i] = fma(b, other, c * qreg[i]);
                }
            }
        } else {
            const bool la = lane < NP && rr + 1 < R;
            LookRead lr;
            if (la) lr = look_load<LD>(st, Mc, cs, sn, rr, lane);
            if (la) {
                double c, s;
                look_finish(lr, skip_tau, c, s);
                cs[rr + 1][lane] = c;
                sn[rr + 1][lane] = s;
            }
        }
        named_bar(bar, QH);
        double* t = Mc;
        Mc = Mn;
        Mn = t;
    }
    if (ltid >= MT && ltid < MT + QT) {
        const int l = (ltid - MT) & 31;
#pragma unroll
        for (int i = 0; i < QR; ++i) Qs[(qrow0 + i) + l * LD] = qreg[i];
    }
    named_bar(bar, QH);
    // Newton-Schulz: Ts <- Q (3I - Q^T Q) / 2 (see solve_pair)
    smem_mma_t<TB, true>(Qs, Qs, Mn, ltid, QH);
    named_bar(bar, QH);
    for (int e = ltid; e < TB * TB; e += QH) {
        const int i = e % TB, j = e / TB;
        Mn[i + j * LD] = (i == j ? 1.5 : 0.0) - 0.5 * Mn[i + j * LD];
    }
    named_bar(bar, QH);
    smem_mma_t<TB, false>(Qs, Mn, Ts, ltid, QH);
    named_bar(bar, QH);
}

// One warp computes a 16 x 32 tile C = A B with K = 32 (m8n8k4 DMMA, 8 k-steps);
// a_at(m, k), b_at(k, n) read the operands, store(m, n, v) writes the result.
template <class FA, class FB, class FC>
__device__ __forceinline__ void warp_tile_16x32(FA a_at, FB b_at, FC store) {
    const int lane = threadIdx.x & 31, r = lane >> 2, kq = lane & 3;
    double acc[2][4][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[mt][t][0] = acc[mt][t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        double af[2], bf[4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) af[mt] = a_at(8 * mt + r, 4 * s + kq);
#pragma unroll
        for (int t = 0; t < 4; ++t) bf[t] = b_at(4 * s + kq, 8 * t + r);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int t = 0; t < 4; ++t) dmma(acc[mt][t][0], acc[mt][t][1], af[mt], bf[t]);
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int i = 0; i < 2; ++i) store(8 * mt + r, 8 * t + 2 * kq + i, acc[mt][t][i]);
}

// One CTA per super-pair of round `round`: composes the round's sub-stages into
// the 64 x 64 rotation Qbuf[pair] (column-major, ld 64); active[pair] = 0 when
// no sub-stage found an entry above skip_tau (Q = I, updates skipped).
__global__ void __launch_bounds__(Q_THREADS, 1)
    jacobi_quad_solve(const double* A, int64_t lda, const SolveTables<32>* tabs, double* Qbuf,
                      int* active, int ns, int round, const double* skip_tau_p, int stage0) {
    extern __shared__ double sm[];
    double* M64 = sm;             // the subproblem, transformed by each sub-stage
    double* Qa = M64 + 64 * L64;  // accumulated 64 x 64 rotation
    double* P = Qa + 64 * L64;    // this sub-stage's two 32 x 32 rotations Q_0, Q_1 (ld L32)
    double* H = P + 64 * L64;     // the halves' solve buffers; Y / Qn temporaries after the solves
    const int tid = threadIdx.x, h = tid >= QH ? 1 : 0, ltid = tid - h * QH;
    double* Mc = H + h * 4 * SUB32;
    double* Mn = Mc + SUB32;
    double* Qs = Mn + SUB32;
    double* csb = H + 8 * SUB32 + h * 2 * 31 * 16;
    auto cs = reinterpret_cast<double(*)[16]>(csb);
    auto sn = reinterpret_cast<double(*)[16]>(csb + 31 * 16);
    auto* st = reinterpret_cast<SolveTables<32>*>(H + 8 * SUB32 + 4 * 31 * 16);
    int a, b;
    circle_pair(ns, round, blockIdx.x, a, b);
    auto g = [&](int i) -> int64_t {
        return i < 32 ? static_cast<int64_t>(a) * 32 + i : static_cast<int64_t>(b) * 32 + (i - 32);
    };
    const bool probe = blockIdx.x == 0 && tid == 0 && round == 5;
    if (probe) SVDK_PROBE_STORE(g_jprobe, 0, SVDK_CLOCK());
    pdl_wait();  // A of the previous round's a64 update (see pdl_trigger)
    const double skip_tau = *skip_tau_p;  // written before the sweep (jacobi_start_kernel)
    for (int e = tid; e < 64 * 64; e += Q_THREADS) {
        const int i = e & 63, j = e >> 6;
        M64[i + j * L64] = __ldcg(&A[g(i) + g(j) * lda]);
        Qa[i + j * L64] = i == j ? 1.0 : 0.0;
    }
    bool any = false;
    const int nsub = stage0 ? 3 : 2;
    for (int s = 0; s < nsub; ++s) {
        const int kind = stage0 ? s : s + 1;
        const int mode = kind == 0 ? 0 : 2;
        const int R = mode == 0 ? 31 : 16;
        {
            const uint4* src = reinterpret_cast<const uint4*>(tabs + mode);
            uint4* dst = reinterpret_cast<uint4*>(st);
            for (int e = tid; e < static_cast<int>(sizeof(SolveTables<32>) / 16); e += Q_THREADS) dst[e] = src[e];
        }
        __syncthreads();  // M64 and the tables ready
        bool big = false;
        for (int e = ltid; e < 32 * 32; e += QH) {
            const int i = e & 31, j = e >> 5;
            const double v = M64[quad_idx(kind, h, i) + quad_idx(kind, h, j) * L64];
            Mc[i + j * L32] = v;
            big |= i != j && fabs(v) > skip_tau;
        }
        const int w0 = __syncthreads_or(big && h == 0);
        const int w1 = __syncthreads_or(big && h == 1);
        if (probe) SVDK_PROBE_STORE(g_jprobe, 1 + 3 * s, SVDK_CLOCK());
        if (!(w0 | w1)) continue;  // uniform: nothing to rotate in this sub-stage
        any = true;
        // each half's rotation Q_h (32 x 32, ld L32) lands in the P region
        quad_sub_solve(Mc, Mn, Qs, P + h * SUB32, *st, cs, sn, R, ltid, 1 + h, h ? w1 != 0 : w0 != 0,
                       skip_tau);
        __syncthreads();
        if (probe) SVDK_PROBE_STORE(g_jprobe, 2 + 3 * s, SVDK_CLOCK());
        // M <- P^T M P and Qa <- Qa P with P = Q_0 (+) Q_1 on the two index
        // sets, as 16 x 32 warp tiles: T1 forms Y_{h1 h2} = M[h1, h2] Q_h2 for
        // the three blocks h1 <= h2 and Qa[:, h] Q_h; T2 forms Q_h1^T Y_{h1 h2},
        // written with its mirror (M stays exactly symmetric).
        const double* Qh = P;
        double* Y = H;                 // Y_00, Y_01, Y_11 (ld L32)
        double* Qn = H + 4 * SUB32;    // Qa[:, h] Q_h: two 64 x 32 (ld L64)
        const int wi = tid >> 5;
        const bool last = s == nsub - 1;  // after the last sub-stage only Qa is needed
        if (wi < 6 && !last) {
            const int blk = wi >> 1, r0 = 16 * (wi & 1);
            const int h1 = blk == 2 ? 1 : 0, h2 = blk == 0 ? 0 : 1;
            warp_tile_16x32(
                [&](int m, int k) { return M64[quad_idx(kind, h1, r0 + m) + quad_idx(kind, h2, k) * L64]; },
                [&](int k, int n) { return Qh[h2 * SUB32 + k + n * L32]; },
                [&](int m, int n, double v) { Y[blk * SUB32 + (r0 + m) + n * L32] = v; });
        } else if (wi < 14) {
            const int hq = (wi - 6) >> 2, r0 = 16 * ((wi - 6) & 3);
            warp_tile_16x32([&](int m, int k) { return Qa[(r0 + m) + quad_idx(kind, hq, k) * L64]; },
                            [&](int k, int n) { return Qh[hq * SUB32 + k + n * L32]; },
                            [&](int m, int n, double v) { Qn[hq * 32 * L64 + (r0 + m) + n * L64] = v; });
        }
        __syncthreads();
        if (wi < 6 && !last) {
            const int blk = wi >> 1, r0 = 16 * (wi & 1);
            const int h1 = blk == 2 ? 1 : 0, h2 = blk == 0 ? 0 : 1;
            warp_tile_16x32([&](int m, int k) { return Qh[h1 * SUB32 + k + (r0 + m) * L32]; },
                            [&](int k, int n) { return Y[blk * SUB32 + k + n * L32]; },
                            [&](int m, int n, double v) {
                                if (h1 == h2 && r0 + m > n) return;
                                const int i = quad_idx(kind, h1, r0 + m), j = quad_idx(kind, h2, n);
                                M64[i + j * L64] = v;
                                M64[j + i * L64] = v;
                            });
        } else {
            const int t0 = last ? 0 : 6 * 32;
            for (int e = tid - t0; e < 64 * 64; e += Q_THREADS - t0) {
                const int row = e & 63, col = (e >> 6) & 31, hq = e >> 11;
                Qa[row + quad_idx(kind, hq, col) * L64] = Qn[hq * 32 * L64 + row + col * L64];
            }
        }
        if (probe && s < 2) SVDK_PROBE_STORE(g_jprobe, 3 + 3 * s, SVDK_CLOCK());
    }
    __syncthreads();
    if (any) {
        double* out = Qbuf + static_cast<size_t>(blockIdx.x) * 4096;
        for (int e = tid; e < 64 * 64; e += Q_THREADS) out[e] = Qa[(e & 63) + (e >> 6) * L64];
    }
    if (tid == 0) active[blockIdx.x] = any ? 1 : 0;
    if (probe) SVDK_PROBE_STORE(g_jprobe, 7, SVDK_CLOCK());
}

// One-sided quad solve (default): the one-sided rounds of jacobi_pair_solve_os
// on the 64 x 64 subproblem. Q (64 x 64, starts at I) and W = M Q (starts at the
// subproblem) only ever see column operations, so the sub-stages compose by
// themselves: a sub-stage is 16 (31 for the in-super-block stage) more rounds
// with another pairing of the 64 columns, and the two-sided 64 x 64 transforms
// between sub-stages of jacobi_quad_solve (and its per-sub-stage Newton-Schulz
// products) disappear. 8 warps: half h = the sub-stage's h-th 32-column
// subproblem, run by 4 warps (16 of the 64 rows each, lane = column) that meet
// at their own named barrier; between sub-stages the columns change hands
// through shared memory. active[pair] = 0 when the subproblem was diagonal to
// skip_tau on entry or no rotation was applied.
constexpr int QOS_THREADS = 256;
constexpr size_t QOS_SMEM = 2 * 64 * L64 * sizeof(double);

template <bool FAST>
__global__ void __launch_bounds__(QOS_THREADS, 1)
    jacobi_quad_solve_os(const double* A, int64_t lda, const SolveTables<32>* tabs, double* Qbuf,
                         int* active, int ns, int round, const double* skip_tau_p, int stage0) {
    constexpr int QR = 16;
    extern __shared__ double sm[];
    double* Qs = sm;
    double* Ws = sm + 64 * L64;
    __shared__ __align__(16) unsigned char sched[2][31][32];  // mode 0, mode 2
    __shared__ double pd[2][2][4][32], px[2][2][4][32];       // [half][buffer][warp][lane]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, h = warp >> 2, w4 = warp & 3;
    const int row0 = QR * w4;
    int a, b;
    circle_pair(ns, round, blockIdx.x, a, b);
    auto g = [&](int i) -> int64_t {
        return i < 32 ? static_cast<int64_t>(a) * 32 + i : static_cast<int64_t>(b) * 32 + (i - 32);
    };
    const bool probe = blockIdx.x == 0 && tid == 0 && round == 5;
    const long long t0 = SVDK_CLOCK();
    {
        constexpr int N16 = 31 * 32 / 16;
        const uint4* s0 = reinterpret_cast<const uint4*>(&tabs[0].part[0][0]);
        const uint4* s2 = reinterpret_cast<const uint4*>(&tabs[2].part[0][0]);
        uint4* dst = reinterpret_cast<uint4*>(&sched[0][0][0]);
        for (int e = tid; e < 2 * N16; e += QOS_THREADS) dst[e] = e < N16 ? s0[e] : s2[e - N16];
    }
    pdl_wait();  // A of the previous round's a64 update
    const double skip_tau = *skip_tau_p;
    const int nsub = stage0 ? 3 : 2;
    int col = quad_idx(stage0 ? 0 : 1, h, lane);  // this lane's column (local 64-index)
    double wreg[QR], qreg[QR];
    bool big = false;
    {
        const double* src = A + g(row0) + g(col) * lda;  // 16 rows inside one super-block
#pragma unroll
        for (int v = 0; v < QR / 4; ++v) {
            const double4 x = ld_cg4(src + 4 * v);
            wreg[4 * v] = x.x; wreg[4 * v + 1] = x.y; wreg[4 * v + 2] = x.z; wreg[4 * v + 3] = x.w;
        }
#pragma unroll
        for (int i = 0; i < QR; ++i) {
            big |= (row0 + i != col) && fabs(wreg[i]) > skip_tau;
            qreg[i] = (row0 + i == col) ? 1.0 : 0.0;
        }
    }
    if (!__syncthreads_or(big)) {  // already diagonal to skip_tau
        if (tid == 0) active[blockIdx.x] = 0;
        return;
    }
    if (probe) {
        SVDK_PROBE_STORE(g_jprobe, 0, t0);
        SVDK_PROBE_STORE(g_jprobe, 1, SVDK_CLOCK());
    }
    bool rotated = false;
    for (int s = 0; s < nsub; ++s) {
        const int kind = stage0 ? s : s + 1;
        if (s > 0) {
            col = quad_idx(kind, h, lane);
#pragma unroll
            for (int i = 0; i < QR; ++i) {
                qreg[i] = Qs[(row0 + i) + col * L64];
                wreg[i] = Ws[(row0 + i) + col * L64];
            }
        }
        const int R = kind == 0 ? 31 : 16;
        rotated |= os_rounds<QR, 4, FAST>(qreg, wreg, sched[kind == 0 ? 0 : 1], R, R, pd[h], px[h], w4, lane,
                                          1 + h, skip_tau);
        if (s + 1 < nsub) {  // the columns change hands
#pragma unroll
            for (int i = 0; i < QR; ++i) {
                Qs[(row0 + i) + col * L64] = qreg[i];
                Ws[(row0 + i) + col * L64] = wreg[i];
            }
            __syncthreads();
        }
        if (probe) SVDK_PROBE_STORE(g_jprobe, 2 + s, SVDK_CLOCK());
    }
    // column-norm Newton step (see jacobi_pair_solve_os); the last sub-stage ran 16 rounds
    double n0 = qreg[0] * qreg[0], n1 = qreg[1] * qreg[1];
#pragma unroll
    for (int i = 2; i < QR; i += 2) {
        n0 = fma(qreg[i], qreg[i], n0);
        n1 = fma(qreg[i + 1], qreg[i + 1], n1);
    }
    pd[h][0][w4][lane] = n0 + n1;
    const bool any = __syncthreads_or(rotated) != 0;
    if (any) {
        const double nn = (pd[h][0][0][lane] + pd[h][0][1][lane]) + (pd[h][0][2][lane] + pd[h][0][3][lane]);
        const double f = fma(-0.5, nn, 1.5);
        double* out = Qbuf + static_cast<size_t>(blockIdx.x) * 4096 + row0 + col * 64;
#pragma unroll
        for (int v = 0; v < QR / 4; ++v)
            st4(out + 4 * v, f * qreg[4 * v], f * qreg[4 * v + 1], f * qreg[4 * v + 2], f * qreg[4 * v + 3]);
    }
    if (tid == 0) active[blockIdx.x] = any ? 1 : 0;
    if (probe) SVDK_PROBE_STORE(g_jprobe, 7, SVDK_CLOCK());
}

// A[ST_p, ST_q] <- Q_p^T A[ST_p, ST_q] Q_q for one super-pair block (p <= q)
// per CTA of 4 warps; X and Q_q are staged in shared memory, warp w computes
// rows [16 w, 16 w + 16) of U = Q_p^T X (its Q_p fragments in registers) and
// then of X' = U Q_q (U re-laid by quad shuffles). X' goes back through shared
// memory with an odd leading dimension (L_OUT = 65), so that both the column
// runs of X' and those of its mirror are read without bank conflicts and
// written to HBM as full 256-byte runs. (Measured alternatives, n = 4096: 8
// warps x 8 rows 114 us, persistent CTAs with a cp.async double buffer and
// Q_q through L1 112 us, this one 105 us.)
constexpr size_t A64_SMEM = 2 * 64 * L64 * sizeof(double);
constexpr int A64_THREADS = 128;
constexpr int L_OUT = 65;

__global__ void __launch_bounds__(A64_THREADS)
    jacobi_update_a64(double* A, int64_t lda, const double* Qbuf, const int* active, int ns, int round) {
    extern __shared__ double sm[];
    double* Xs = sm;
    double* Qs = sm + 64 * L64;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, r = lane >> 2, kq = lane & 3;
    const int u = blockIdx.x;
    pdl_wait();  // Q and the active flags of this round's quad solve
    int q = static_cast<int>((sqrt(8.0 * u + 1.0) - 1.0) * 0.5);
    while ((q + 1) * (q + 2) / 2 <= u) ++q;
    while (q * (q + 1) / 2 > u) --q;
    const int p = u - q * (q + 1) / 2;
    const bool ap = __ldcg(&active[p]) != 0, aq = __ldcg(&active[q]) != 0;
    if (!(ap | aq)) return;
    int pa, pb, qa, qb;
    circle_pair(ns, round, p, pa, pb);
    circle_pair(ns, round, q, qa, qb);
    auto gp = [&](int i) -> int64_t {
        return i < 32 ? static_cast<int64_t>(pa) * 32 + i : static_cast<int64_t>(pb) * 32 + (i - 32);
    };
    auto gq = [&](int i) -> int64_t {
        return i < 32 ? static_cast<int64_t>(qa) * 32 + i : static_cast<int64_t>(qb) * 32 + (i - 32);
    };
    const double* Qp = Qbuf + static_cast<size_t>(p) * 4096;
    const double* Qq = Qbuf + static_cast<size_t>(q) * 4096;
#pragma unroll 8
    for (int it = 0; it < 2048 / A64_THREADS; ++it) {
        const int e = tid + it * A64_THREADS;
        const int i = (e & 31) * 2, j = e >> 5;
        const double2 x = __ldcg(reinterpret_cast<const double2*>(&A[gp(i) + gq(j) * lda]));
        // the rotation slots are read beside the active flags, not behind them (always allocated)
        double2 y = __ldcg(reinterpret_cast<const double2*>(&Qq[i + j * 64]));
        if (!aq) y = make_double2(i == j ? 1.0 : 0.0, i + 1 == j ? 1.0 : 0.0);
        *reinterpret_cast<double2*>(&Xs[i + j * L64]) = x;
        *reinterpret_cast<double2*>(&Qs[i + j * L64]) = y;
    }
    // A-fragments of Q_p^T: (Q_p^T)[m][k] = Q_p[k][m], m = 16 w + 8 mt + r, k = 4 s + kq
    double qpf[16][2];
#pragma unroll
    for (int s = 0; s < 16; ++s)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            const int k = 4 * s + kq, m = 16 * w + 8 * mt + r;
            qpf[s][mt] = __ldcg(&Qp[k + m * 64]);
            if (!ap) qpf[s][mt] = k == m ? 1.0 : 0.0;
        }
    __syncthreads();
    double U[2][8][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int t = 0; t < 8; ++t) U[mt][t][0] = U[mt][t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        double bx[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) bx[t] = Xs[(4 * s + kq) + (8 * t + r) * L64];
#pragma unroll
        for (int t = 0; t < 8; ++t)
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) dmma(U[mt][t][0], U[mt][t][1], qpf[s][mt], bx[t]);
    }
    double O[2][8][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int t = 0; t < 8; ++t) O[mt][t][0] = O[mt][t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        // U[8 mt + r][4 s + kq] lives in lane (r, 2 (s & 1) + kq / 2), register U[mt][s / 2][kq & 1]
        const int src = (lane & ~3) | (2 * (s & 1) + (kq >> 1));
        double bq[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) bq[t] = Qs[(4 * s + kq) + (8 * t + r) * L64];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            const double v0 = __shfl_sync(0xffffffffu, U[mt][s >> 1][0], src);
            const double v1 = __shfl_sync(0xffffffffu, U[mt][s >> 1][1], src);
            const double av = (kq & 1) ? v1 : v0;
#pragma unroll
            for (int t = 0; t < 8; ++t) dmma(O[mt][t][0], O[mt][t][1], av, bq[t]);
        }
    }
    __syncthreads();  // every warp is done reading Xs
    double* Xo = Xs;  // X' with leading dimension L_OUT
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int t = 0; t < 8; ++t)
#pragma unroll
            for (int i = 0; i < 2; ++i) Xo[(16 * w + 8 * mt + r) + (8 * t + 2 * kq + i) * L_OUT] = O[mt][t][i];
    __syncthreads();
    if (p == q) {  // diagonal super-pair block: upper triangle mirrored (exact symmetry)
#pragma unroll 4
        for (int e = tid; e < 4096; e += A64_THREADS) {
            const int i = e & 63, j = e >> 6;
            A[gp(i) + gp(j) * lda] = i <= j ? Xo[i + j * L_OUT] : Xo[j + i * L_OUT];
        }
        return;
    }
#pragma unroll 4
    for (int e = tid; e < 4096; e += A64_THREADS) {  // X': lanes walk a column of X'
        const int i = e & 63, j = e >> 6;
        A[gp(i) + gq(j) * lda] = Xo[i + j * L_OUT];
    }
#pragma unroll 4
    for (int e = tid; e < 4096; e += A64_THREADS) {  // mirror: lanes walk a row of X'
        const int jj = e & 63, ii = e >> 6;
        A[gq(jj) + gp(ii) * lda] = Xo[ii + jj * L_OUT];
    }
}

// V[rows, ST_q] <- V[rows, ST_q] Q_q: one CTA of 4 warps per (super-pair q,
// V64_ROWS-row chunk), Q_q staged in shared memory; a warp walks 16-row tiles
// with the rows permuted so that m8n8k4 row r of m-tile m is tile row 2 r + m
// (each lane owns 2 consecutive rows: every V access is a 16-byte LDG/STG and
// 8 lanes cover a full 128-byte column run). Four CTAs per SM keep loads of
// one warp in flight under the DMMAs of the others.
constexpr int V64_ROWS = 256;

__global__ void __launch_bounds__(128, 4)
    jacobi_update_v64(double* V, int64_t ldv, int64_t n_rows, const double* Qbuf, const int* active,
                      int ns, int round) {
    __shared__ double Qs[64 * L64];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, r = lane >> 2, kq = lane & 3;
    const int ks = ns / 2;
    const int q = static_cast<int>(blockIdx.x % ks);
    const int64_t row_begin = static_cast<int64_t>(blockIdx.x / ks) * V64_ROWS;
    if (row_begin >= n_rows || !__ldcg(&active[q])) return;
    int qa, qb;
    circle_pair(ns, round, q, qa, qb);
    const double* Qq = Qbuf + static_cast<size_t>(q) * 4096;
#pragma unroll
    for (int it = 0; it < 16; ++it) {
        const int e = tid + it * 128;
        const int i = (e & 31) * 2, j = e >> 5;
        const double2 y = __ldcg(reinterpret_cast<const double2*>(&Qq[i + j * 64]));
        Qs[i + j * L64] = y.x;
        Qs[i + 1 + j * L64] = y.y;
    }
    const int64_t row_end = min(n_rows, row_begin + V64_ROWS);
    // column bases: k-step s reads column gq(4 s + kq), t-tile stores gq(8 t + 2 kq + i)
    const int64_t step = 4 * ldv;
    const double* ca = V + 2 * r + (static_cast<int64_t>(qa) * 32 + kq) * ldv;
    const double* cb = V + 2 * r + (static_cast<int64_t>(qb) * 32 + kq) * ldv;
    double* sa = V + 2 * r + (static_cast<int64_t>(qa) * 32 + 2 * kq) * ldv;
    double* sb = V + 2 * r + (static_cast<int64_t>(qb) * 32 + 2 * kq) * ldv;
    __syncthreads();
    for (int64_t row0 = row_begin + 16 * w; row0 < row_end; row0 += 64) {
        double2 va[16];
#pragma unroll
        for (int s = 0; s < 16; ++s) va[s] = ld_cg2((s < 8 ? ca : cb) + row0 + (s & 7) * step);
        double acc[2][8][2];
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int t = 0; t < 8; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            double bq[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) bq[t] = Qs[(4 * s + kq) + (8 * t + r) * L64];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                dmma(acc[0][t][0], acc[0][t][1], va[s].x, bq[t]);
                dmma(acc[1][t][0], acc[1][t][1], va[s].y, bq[t]);
            }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t)
#pragma unroll
            for (int i = 0; i < 2; ++i)
                *reinterpret_cast<double2*>((t < 4 ? sa : sb) + row0 + (t & 3) * 2 * step + i * ldv) =
                    make_double2(acc[0][t][i], acc[1][t][i]);
    }
}

void build_quad_plan(Ctx* c, JacobiPlan& P) {
    const int64_t n_pad = P.n_pad;
    const int ns = static_cast<int>(n_pad / 32), ks = ns / 2, rounds = ns - 1;
    ensure_smem_attr(reinterpret_cast<const void*>(jacobi_quad_solve), QUAD_SMEM);
    ensure_smem_attr(reinterpret_cast<const void*>(jacobi_quad_solve_os<true>), QOS_SMEM);
    ensure_smem_attr(reinterpret_cast<const void*>(jacobi_quad_solve_os<false>), QOS_SMEM);
    ensure_smem_attr(reinterpret_cast<const void*>(jacobi_update_a64), A64_SMEM);
    // SVDK_JACOBI_OS=0: the two-sided quad solve; SVDK_JACOBI_FASTROT=0: rsqrt()-based rotation
    const char* os_env = std::getenv("SVDK_JACOBI_OS");
    const bool qos = !(os_env && std::atoi(os_env) == 0);
    const char* fast_env = std::getenv("SVDK_JACOBI_FASTROT");
    const bool os_fast = !(fast_env && std::atoi(fast_env) == 0);
    P.qbuf = DBuf(c, static_cast<size_t>(rounds) * ks * 4096);
    P.act = DBuf(c, static_cast<size_t>(rounds) * ks);
    int* active = reinterpret_cast<int*>(P.act.p());
    if (!c->aux_stream) {
        SVDK_CUDA(cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
        SVDK_CUDA(cudaEventCreateWithFlags(&c->aux_ev[0], cudaEventDisableTiming));
        SVDK_CUDA(cudaEventCreateWithFlags(&c->aux_ev[1], cudaEventDisableTiming));
    }
    cudaStream_t S = c->stream;
    P.tabs = DBuf(c, 3 * sizeof(SolveTables<32>) / sizeof(double));
    jacobi_tables_kernel<32><<<3, 256, 0, S>>>(reinterpret_cast<SolveTables<32>*>(P.tabs.p()));
    SVDK_CHECK_LAUNCH();
    c->launches++;
    const auto* tabs = reinterpret_cast<const SolveTables<32>*>(P.tabs.p());
    const int a_ctas = ks * (ks + 1) / 2;
    const int v_ctas = static_cast<int>(ceil_div(n_pad, static_cast<int64_t>(V64_ROWS))) * ks;
    // solve -> a64 -> solve as programmatic dependent launches (see pdl_trigger)
    const char* pdl_env = std::getenv("SVDK_JACOBI_PDL");
    const bool pdl = !(pdl_env && std::atoi(pdl_env) == 0);
    double* A = P.A.p();
    double* V = P.V.p();
    const double* skip_p = P.scal.p() + JS_SKIP;
    double* qbase = P.qbuf.p();
    P.launches_per_sweep = 3 * rounds;
    P.enqueue_sweep = [=]() {
        const cudaStream_t S = c->stream, S2 = c->aux_stream;
        const cudaEvent_t ev0 = c->aux_ev[0], ev1 = c->aux_ev[1];
        const double* a_in = A;
        int64_t ld = n_pad;
        auto launch = [&](auto kern, int grid, int block, size_t smem, auto... args) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(static_cast<unsigned>(grid));
            cfg.blockDim = dim3(static_cast<unsigned>(block));
            cfg.dynamicSmemBytes = smem;
            cfg.stream = S;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = pdl ? 1 : 0;
            SVDK_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
        };
        for (int r = 0; r < rounds; ++r) {
            double* qr = qbase + static_cast<size_t>(r) * ks * 4096;
            int* ar = active + static_cast<size_t>(r) * ks;
            if (qos)
                launch(os_fast ? jacobi_quad_solve_os<true> : jacobi_quad_solve_os<false>, ks, QOS_THREADS, QOS_SMEM,
                       a_in, ld, tabs, qr, ar, ns, r, skip_p, r == 0 ? 1 : 0);
            else
                launch(jacobi_quad_solve, ks, Q_THREADS, QUAD_SMEM, a_in, ld, tabs, qr, ar, ns, r, skip_p,
                       r == 0 ? 1 : 0);
            SVDK_CUDA(cudaEventRecord(ev0, S));
            SVDK_CUDA(cudaStreamWaitEvent(S2, ev0, 0));
            jacobi_update_v64<<<v_ctas, 128, 0, S2>>>(V, n_pad, n_pad, qr, ar, ns, r);
            const double* qc = qr;
            const int* ac = ar;
            launch(jacobi_update_a64, a_ctas, A64_THREADS, A64_SMEM, A, ld, qc, ac, ns, r);
        }
        SVDK_CUDA(cudaEventRecord(ev1, S2));
        SVDK_CUDA(cudaStreamWaitEvent(S, ev1, 0));
    };
    build_loop_graph(c, P);
}

}  // namespace

// Smallest n that uses the quad scheme by default. Measured on B200
// (tools/eig_time.py with SVDK_JACOBI_TB, Gram spectra, one-sided solves): n = 1536 / 2048 / 2560 /
// 3072 take 26.0 / 45.7 / 100.0 / 167.6 ms with 2b = 32 and 29.2 / 48.7 / 85.4 / 142.1 ms with the
// quad scheme — below n ~ 2300 the solve chain (not the update traffic) bounds a sweep.
constexpr int64_t kQuadMinN = 2304;

// The context's sweep plan for (n_pad, TB), built on first use and kept
// (most recently used last, at most kMaxPlans per context).
JacobiPlan& jacobi_plan(Ctx* c, int64_t n_pad, int TB) {
    if (!c->jacobi_cache) c->jacobi_cache = new JacobiCache;
    auto& plans = c->jacobi_cache->plans;
    for (size_t i = 0; i < plans.size(); ++i)
        if (plans[i]->n_pad == n_pad && plans[i]->tb == TB && plans[i]->A.count()) {
            std::unique_ptr<JacobiPlan> p = std::move(plans[i]);
            plans.erase(plans.begin() + static_cast<long>(i));
            plans.push_back(std::move(p));
            return *plans.back();
        }
    if (plans.size() >= kMaxPlans) plans.erase(plans.begin());
    auto p = std::make_unique<JacobiPlan>();
    p->n_pad = n_pad;
    p->tb = TB;
    p->A = DBuf(c, static_cast<size_t>(n_pad) * n_pad);
    p->V = DBuf(c, static_cast<size_t>(n_pad) * n_pad);
    p->blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(n_pad, 2 * c->num_sms)));  // column-strided sumsq
    p->part_all = DBuf(c, 2 * static_cast<size_t>(std::max<int64_t>(p->blocks, 2 * c->num_sms)));
    p->part_low = DBuf(c, static_cast<size_t>(p->blocks));
    p->scal = DBuf(c, JS_COUNT);
    fill(c, p->scal.p(), JS_COUNT, 0.0);
    JacobiPlan& P = *p;
    plans.push_back(std::move(p));
    std::lock_guard<std::mutex> lock(graph_mutex());
    try {
        if (TB == 16)
            build_pair_plan<16>(c, P);
        else if (TB == 64)
            build_quad_plan(c, P);
        else
            build_pair_plan<32>(c, P);
    } catch (...) {
        plans.pop_back();
        throw;
    }
    return P;
}

void eig_sym(Ctx* c, const double* S, int64_t lds, int64_t n, int max_sweeps, double* w,
             double* Vout, int64_t ldv) {
    if (max_sweeps <= 0) max_sweeps = 30;
    if (n == 0) return;
    PhaseTimer timer(c, "eig_sym");
    // Block size: measured on B200 (tools/eig_sweep.sh): 2b = 32 with ONE
    // inner sweep per round is fastest for n in [256, 2048]; the outer sweep
    // count (9-12) does not depend on how far each subproblem is pushed.
    // TB = 64: the quad scheme (64-wide updates, section 3 above) for large n,
    // where the per-round A/V updates dominate.
    int TB = n <= 64 ? 16 : (n >= kQuadMinN ? 64 : 32);
    if (const char* e = std::getenv("SVDK_JACOBI_TB")) {  // tuning override
        const int t = std::atoi(e);
        if (t == 16 || t == 32 || t == 64) TB = t;
    }
    const int64_t n_pad = round_up(n, TB);
    JacobiPlan& P = jacobi_plan(c, n_pad, TB);
    double* scal = P.scal.p();
    // symmetry check + prescale on the device (kernels.cpp:251-269); the
    // ParamError is raised after the single read-back at the end
    {
        const int blocks = static_cast<int>(
            std::max<int64_t>(1, std::min<int64_t>(ceil_div(n * n, 256), 2 * c->num_sms)));
        symcheck_kernel<<<blocks, 256, 0, c->stream>>>(S, lds, n, P.part_all.p());
        const char* pe = std::getenv("SVDK_JACOBI_POLISH");
        const int polish = !(pe && std::atoi(pe) == 0);
        eig_prep_kernel<<<1, 32, 0, c->stream>>>(P.part_all.p(), blocks, max_sweeps, polish, scal);
        const int iblocks = static_cast<int>(
            std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_pad * n_pad, 256), 4 * c->num_sms)));
        jacobi_init_kernel<<<iblocks, 256, 0, c->stream>>>(S, lds, n, P.A.p(), P.V.p(), n_pad, scal + JS_SCALE);
        SVDK_CHECK_LAUNCH();
        c->launches += 3;
    }
    int sweeps = run_plan(c, P);
    DBuf dest(c, n);  // int storage inside a double buffer
    eig_sort_kernel<<<static_cast<unsigned>(ceil_div(n, 128)), 128, 0, c->stream>>>(
        P.A.p(), n_pad, n, scal + JS_UNSCALE, w, reinterpret_cast<int*>(dest.p()));
    SVDK_CHECK_LAUNCH();
    dim3 g(static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 128), 64)),
           static_cast<unsigned>(std::min<int64_t>(n, 65535)));
    eig_gather_kernel<<<g, 128, 0, c->stream>>>(P.V.p(), n_pad, n,
                                                reinterpret_cast<const int*>(dest.p()), Vout, ldv);
    SVDK_CHECK_LAUNCH();
    c->launches += 2;
    double h[JS_COUNT];
    d2h(c, h, scal, JS_COUNT);
    if (sweeps < 0) {
        sweeps = static_cast<int>(h[JS_SWEEPS]);
        const int executed = sweeps + (h[JS_POLISH] == 2.0 ? 1 : 0);
        c->launches += static_cast<int64_t>(executed) * (P.launches_per_sweep + 2) + 3;
    }
    if (h[JS_MASYM] > 1e-8 * h[JS_MABS]) {
        char buf[96];
        std::snprintf(buf, sizeof buf, "%f", h[JS_MASYM]);
        fail(SVDK_E_PARAM, std::string("eig_sym: input asymmetric beyond tolerance, max|s-s^T| = ") + buf);
    }
    c->jacobi_sweeps = sweeps;
    const double off = h[JS_OFF] * h[JS_UNSCALE];  // back to the caller's units
    c->last_off_norm = off;
    if (off > h[JS_THR] * h[JS_UNSCALE]) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "eig_sym: no convergence in %d sweeps, off-diagonal norm %f",
                      max_sweeps, off);
        fail(SVDK_E_NUMERICAL, buf, off);
    }
}

void jacobi_cache_free(Ctx* c) {
    delete c->jacobi_cache;
    c->jacobi_cache = nullptr;
}

}  // namespace svdk

extern "C" int svdk_debug_jacobi_timeline(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, svdk::g_jtimeline, 16 * 8 * sizeof(unsigned long long)) == cudaSuccess ? 0 : 4;
}

extern "C" int svdk_debug_jacobi_probe(long long* out) {
    return cudaMemcpyFromSymbol(out, svdk::g_jprobe, 16 * sizeof(long long)) == cudaSuccess ? 0 : 4;
}
