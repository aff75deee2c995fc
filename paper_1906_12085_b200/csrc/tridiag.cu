// tridiag.cu — eigenpairs of the Lanczos tridiagonal T = tridiag(beta, alpha, beta)
// in O(k^2) work (k = Lanczos steps), replacing the dense k x k Jacobi on T.
//
//   eigenvalues   warp-per-eigenvalue multisection on Sturm counts (LAPACK
//                 dstebz's recurrence with the pivmin guard): each iteration a
//                 warp evaluates 32 points of its interval, ~5 bits per
//                 iteration, to |width| <= 2 eps max(|lo|, |hi|);
//   eigenvectors  thread-per-eigenvector twisted factorisation (the core of
//                 MRRR's dlar1v): T - lambda I = L D L^T (top-down) and
//                 U P U^T (bottom-up), twist index r = argmin |gamma_r|,
//                 x_r = 1 and the two one-sided recurrences;
//   orthonormality S^T S = I to 1e-6 certifies the basis, one Newton-Schulz
//                 polar step S (3I - S^T S)/2 (two DMMA products) polishes it.
// Tight clusters (relative gap < 1e-10) and a failed certification return
// false: the caller then solves T densely with the Jacobi eigensolver. The
// Lanczos T of BASELINE's configs has relative gaps >= ~1e-7.
#include <cfloat>

#include "svdk_methods.h"

namespace svdk {
namespace {

constexpr int TB_THREADS = 256;   // setup kernel
constexpr int BIS_WARPS = 8;      // eigenvalues per bisection CTA
constexpr int VEC_THREADS = 128;  // eigenvectors per vector CTA

// info: [0] lo, [1] hi (Gershgorin), [2] pivmin, [3] max |lambda| bound
__global__ void __launch_bounds__(TB_THREADS)
    tri_setup_kernel(const double* alpha, const double* beta, int n, double* b2, double* info) {
    __shared__ double rlo[TB_THREADS / 32], rhi[TB_THREADS / 32], rb[TB_THREADS / 32];
    double lo = DBL_MAX, hi = -DBL_MAX, bmax = 0.0;
    for (int i = threadIdx.x; i < n; i += TB_THREADS) {
        const double bl = i > 0 ? fabs(beta[i - 1]) : 0.0, br = i + 1 < n ? fabs(beta[i]) : 0.0;
        lo = fmin(lo, alpha[i] - bl - br);
        hi = fmax(hi, alpha[i] + bl + br);
        if (i + 1 < n) {
            const double bb = beta[i] * beta[i];
            b2[i] = bb;
            bmax = fmax(bmax, bb);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        bmax = fmax(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) rlo[w] = lo, rhi[w] = hi, rb[w] = bmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < TB_THREADS / 32; ++k) {
            lo = fmin(lo, rlo[k]);
            hi = fmax(hi, rhi[k]);
            bmax = fmax(bmax, rb[k]);
        }
        const double tnorm = fmax(fabs(lo), fabs(hi));
        // widen the Gershgorin interval slightly (dstebz) so it strictly contains the spectrum
        const double pad = 2.0 * DBL_EPSILON * tnorm * n + 2.0 * DBL_MIN;
        info[0] = lo - pad;
        info[1] = hi + pad;
        info[2] = DBL_MIN * fmax(1.0, bmax);
        info[3] = tnorm;
    }
}

// number of eigenvalues of T strictly below x (Sturm count, dstebz guard)
template <bool kShared>
__device__ __forceinline__ int sturm_count(const double* a, const double* b2, int n, double x, double pivmin) {
    double q = a[0] - x;
    if (fabs(q) <= pivmin) q = -pivmin;
    int cnt = q < 0.0;
    for (int i = 1; i < n; ++i) {
        q = (a[i] - x) - b2[i - 1] / q;
        if (fabs(q) <= pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

// warp w of the grid finds the (k-1-w)-th smallest = w-th largest eigenvalue
template <bool kShared>
__global__ void __launch_bounds__(BIS_WARPS * 32)
    tri_bisect_kernel(const double* alpha, const double* b2g, int n, const double* info, double* w_desc) {
    extern __shared__ double sh[];
    const double* a = alpha;
    const double* b2 = b2g;
    if (kShared) {
        double* sa = sh;
        double* sb = sh + n;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            sa[i] = alpha[i];
            if (i + 1 < n) sb[i] = b2g[i];
        }
        __syncthreads();
        a = sa;
        b2 = sb;
    }
    const int lane = threadIdx.x & 31;
    const int wi = blockIdx.x * BIS_WARPS + (threadIdx.x >> 5);
    if (wi >= n) return;
    const int idx = n - 1 - wi;  // ascending index of the wi-th largest eigenvalue
    const double pivmin = info[2];
    double lo = info[0], hi = info[1];
    for (int it = 0; it < 40; ++it) {
        const double width = hi - lo;
        if (width <= fmax(2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)), 4.0 * pivmin)) break;
        const double x = fma(width, static_cast<double>(lane + 1) / 33.0, lo);
        const int cnt = sturm_count<kShared>(a, b2, n, x, pivmin);
        const unsigned above = __ballot_sync(0xffffffffu, cnt > idx);  // lambda_idx < x
        const int f = above ? __ffs(above) - 1 : 32;                  // first point above
        const double xf = __shfl_sync(0xffffffffu, x, f & 31);
        const double xp = __shfl_sync(0xffffffffu, x, (f + 31) & 31);
        if (f < 32) hi = xf;
        if (f > 0) lo = xp;
    }
    if (lane == 0) w_desc[wi] = 0.5 * (lo + hi);
}

// thread t computes the eigenvector of w_desc[t] by the twisted factorisation.
// Scratch is interleaved by eigenvector (element i of vector t at [i * n + t])
// so a warp's accesses are coalesced: X ends as S^T (column-major n x n with
// the eigenvector index as the row), U holds the u multipliers.
__global__ void __launch_bounds__(VEC_THREADS)
    tri_vec_kernel(const double* alpha, const double* beta, int n, const double* info, const double* w_desc,
                   double* X, double* U) {
    const int t = blockIdx.x * VEC_THREADS + threadIdx.x;
    if (t >= n) return;
    const double lam = w_desc[t], pivmin = info[2];
    const int64_t ld = n;
    // stationary: T - lam I = L D L^T, d_0 = a_0 - lam, d_{i+1} = a_{i+1} - lam - b_i^2 / d_i
    double d = alpha[0] - lam;
    if (fabs(d) <= pivmin) d = -pivmin;
    X[t] = d;
    for (int i = 0; i + 1 < n; ++i) {
        d = (alpha[i + 1] - lam) - beta[i] * (beta[i] / d);
        if (fabs(d) <= pivmin) d = -pivmin;
        X[(i + 1) * ld + t] = d;
    }
    // progressive: T - lam I = U P U^T from the bottom, gamma_i = d_i + p_i - (a_i - lam)
    double p = alpha[n - 1] - lam;
    if (fabs(p) <= pivmin) p = -pivmin;
    int r = n - 1;
    double gbest = fabs(X[(n - 1) * ld + t] + p - (alpha[n - 1] - lam));
    for (int i = n - 2; i >= 0; --i) {
        const double ui = beta[i] / p;  // u_i = b_i / p_{i+1}
        U[i * ld + t] = ui;
        p = (alpha[i] - lam) - beta[i] * ui;
        if (fabs(p) <= pivmin) p = -pivmin;
        const double g = fabs(X[i * ld + t] + p - (alpha[i] - lam));
        if (g < gbest) gbest = g, r = i;
    }
    // x_r = 1; upward x_i = -(b_i / d_i) x_{i+1}; downward x_{i+1} = -u_i x_i
    double nrm = 1.0;
    double xv = 1.0;
    for (int i = r - 1; i >= 0; --i) {
        xv = -(beta[i] / X[i * ld + t]) * xv;
        X[i * ld + t] = xv;
        nrm = fma(xv, xv, nrm);
    }
    X[r * ld + t] = 1.0;
    xv = 1.0;
    for (int i = r; i + 1 < n; ++i) {
        xv = -U[i * ld + t] * xv;
        X[(i + 1) * ld + t] = xv;
        nrm = fma(xv, xv, nrm);
    }
    const double inv = rsqrt(nrm);
    for (int i = 0; i < n; ++i) X[i * ld + t] *= inv;
}

// B = (3 I - G) / 2 for one Newton-Schulz polar step S <- S B (G = S^T S);
// flag |= 2 when G is not I to 1e-6 (the twisted-factorisation vectors were
// not numerically orthogonal: unresolved cluster).
__global__ void tri_ns_kernel(const double* G, int n, double* Bm, int* flag) {
    const int64_t nn = static_cast<int64_t>(n) * n;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nn;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / n, i = e - j * n;
        const double d = G[e] - (i == j ? 1.0 : 0.0);
        if (!(fabs(d) <= 1e-6)) atomicOr(flag, 2);
        Bm[e] = (i == j ? 1.0 : 0.0) - 0.5 * d;
    }
}

// flag = 1 when two neighbouring eigenvalues are closer than 1e-10 ||T|| (or non-finite)
__global__ void tri_gap_kernel(const double* w_desc, int n, const double* info, int* flag) {
    const double tol = 1e-10 * fmax(info[3], DBL_MIN);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double a = w_desc[i];
        if (!isfinite(a) || (i + 1 < n && !(a - w_desc[i + 1] > tol))) atomicOr(flag, 1);
    }
}

}  // namespace

// Eigenpairs of the symmetric tridiagonal T (alpha k, beta k-1) on the device:
// w (k, descending), S (k x k, lds >= k, even) orthonormal eigenvectors.
// Returns false (w, S unspecified) when T has eigenvalue clusters the O(k^2)
// path does not resolve; the caller then uses the dense eigensolver.
bool tridiag_eig(Ctx* c, const double* alpha, const double* beta, int64_t k, double* w, double* S, int64_t lds) {
    if (k <= 0) return true;
    if (k > (int64_t(1) << 30) || lds < k || lds % 2) return false;
    const int n = static_cast<int>(k);
    PhaseTimer timer(c, "tridiag_eig", 0.0, 0.0);
    DBuf b2(c, std::max<int64_t>(k, 1)), info(c, 4), flag(c, 1);
    SVDK_CUDA(cudaMemsetAsync(flag.p(), 0, sizeof(double), c->stream));
    tri_setup_kernel<<<1, TB_THREADS, 0, c->stream>>>(alpha, beta, n, b2.p(), info.p());
    SVDK_CHECK_LAUNCH();
    const unsigned bgrid = static_cast<unsigned>(ceil_div(k, BIS_WARPS));
    const size_t smem = 2 * sizeof(double) * static_cast<size_t>(k);
    if (smem <= 200 * 1024) {
        ensure_smem_attr(reinterpret_cast<const void*>(tri_bisect_kernel<true>), smem);
        tri_bisect_kernel<true><<<bgrid, BIS_WARPS * 32, smem, c->stream>>>(alpha, b2.p(), n, info.p(), w);
    } else {
        tri_bisect_kernel<false><<<bgrid, BIS_WARPS * 32, 0, c->stream>>>(alpha, b2.p(), n, info.p(), w);
    }
    SVDK_CHECK_LAUNCH();
    int* fl = reinterpret_cast<int*>(flag.p());
    tri_gap_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(k, 256), 1024)), 256, 0, c->stream>>>(
        w, n, info.p(), fl);
    SVDK_CHECK_LAUNCH();
    c->launches += 3;
    int bad = 0;
    SVDK_CUDA(cudaMemcpyAsync(&bad, fl, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    SVDK_CUDA(cudaStreamSynchronize(c->stream));
    if (bad) return false;
    {
        DBuf X(c, static_cast<size_t>(k) * k), Us(c, static_cast<size_t>(k) * k);
        tri_vec_kernel<<<static_cast<unsigned>(ceil_div(k, VEC_THREADS)), VEC_THREADS, 0, c->stream>>>(
            alpha, beta, n, info.p(), w, X.p(), Us.p());
        SVDK_CHECK_LAUNCH();
        c->launches++;
        Us.reset();
        DBuf S0(c, static_cast<size_t>(lds) * k), G(c, static_cast<size_t>(k) * k), Bm(c, static_cast<size_t>(k) * k);
        transpose(c, X.p(), k, k, k, S0.p(), lds);
        X.reset();
        // certify (S0^T S0 = I to 1e-6) and polish by one Newton-Schulz step
        // S = S0 (3 I - S0^T S0) / 2: orthogonality 1e-12 -> rounding level,
        // order and signs kept (two DMMA products instead of a CholeskyQR2)
        syrk(c, k, k, S0.p(), lds, G.p(), k);
        tri_ns_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(k * k, 256), 4096)), 256, 0, c->stream>>>(
            G.p(), n, Bm.p(), fl);
        SVDK_CHECK_LAUNCH();
        c->launches++;
        gemm(c, false, k, k, k, S0.p(), lds, Bm.p(), k, S, lds);
        SVDK_CUDA(cudaMemcpyAsync(&bad, fl, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        SVDK_CUDA(cudaStreamSynchronize(c->stream));
        if (bad) return false;
    }
    return true;
}

}  // namespace svdk
