// synth.h — the seeded synthetic-input generator of SURVEY §8d, bit-identical
// on the host CPU and on the GPU (shared by bench.py, the tests and the
// golden-fixture scripts; NOT on the PCA path).
//
// Every Gaussian is a pure function of (seed, stream, global element index):
//   counter-based Philox4x32-10 -> two 53-bit uniforms -> Box-Muller, with log
//   and sin/cos evaluated by fixed polynomials written with explicitly rounded
//   operations (__dadd_rn/__dmul_rn/__fma_rn/__ddiv_rn/__dsqrt_rn on the
//   device, the same IEEE operations with -ffp-contract=off on the host). So a
//   row shard generated on rank r of N is byte-identical to the same rows of
//   the N = 1 matrix, and to what the fixture scripts generate on the CPU.
//
// The matrix is A = X M + sigma N (BASELINE.json configs):
//   X (m x n)  Gaussians quantised to multiples of 2^-10 (|x| < 16), stream 1;
//   M (n x n)  = R_X^-1 diag(s) V0^T, quantised to a fixed-point grid, where
//              R_X = chol(X^T X) (so U0 = X R_X^-1 has orthonormal columns)
//              and V0 = CholeskyQR2 of a quantised n x n Gaussian (stream 2);
//   N (m x n)  Gaussians, stream 3.
// The quantisation makes X^T X and X M EXACT in fp64 whatever the summation
// order (every partial sum is an integer multiple of the grid below 2^53), so
// the DMMA GEMMs on the GPU, numpy on the CPU and an NCCL allreduce of
// per-rank partial Grams all produce the same bits. The quantisation perturbs
// the designed signal by ~2^-27 relative — far below every config's noise.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define SY_HD __host__ __device__ __forceinline__
#else
#define SY_HD static inline
#include <math.h>
#endif

#if defined(__CUDA_ARCH__)
#define SY_ADD(a, b) __dadd_rn((a), (b))
#define SY_SUB(a, b) __dsub_rn((a), (b))
#define SY_MUL(a, b) __dmul_rn((a), (b))
#define SY_FMA(a, b, c) __fma_rn((a), (b), (c))
#define SY_DIV(a, b) __ddiv_rn((a), (b))
#define SY_SQRT(a) __dsqrt_rn((a))
#define SY_RINT(a) rint((a))
#else
// host: compiled with -ffp-contract=off (no implicit fma), fma() is the
// correctly rounded C99 fused multiply-add.
#define SY_ADD(a, b) ((a) + (b))
#define SY_SUB(a, b) ((a) - (b))
#define SY_MUL(a, b) ((a) * (b))
#define SY_FMA(a, b, c) fma((a), (b), (c))
#define SY_DIV(a, b) ((a) / (b))
#define SY_SQRT(a) sqrt((a))
#define SY_RINT(a) nearbyint((a))
#endif

enum { SY_STREAM_X = 1, SY_STREAM_V = 2, SY_STREAM_NOISE = 3 };

// X is quantised to multiples of 2^-SY_XBITS with |x| <= SY_XMAX * 2^-SY_XBITS.
#define SY_XBITS 10
#define SY_XMAX 16383.0

SY_HD uint32_t sy_mulhilo(uint32_t a, uint32_t b, uint32_t* hi) {
    const uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    return (uint32_t)p;
}

// Philox4x32-10 (Salmon et al., SC'11): counter c, key k.
SY_HD void sy_philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, hi1;
        const uint32_t lo0 = sy_mulhilo(0xD2511F53u, c[0], &hi0);
        const uint32_t lo1 = sy_mulhilo(0xCD9E8D57u, c[2], &hi1);
        const uint32_t n0 = hi1 ^ c[1] ^ k0;
        const uint32_t n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

SY_HD double sy_u64_as_double(uint64_t u) {
    union {
        uint64_t u;
        double d;
    } x;
    x.u = u;
    return x.d;
}
SY_HD uint64_t sy_double_as_u64(double d) {
    union {
        uint64_t u;
        double d;
    } x;
    x.d = d;
    return x.u;
}

// Natural log of x in [2^-53, 1] (the Box-Muller radius argument).
// x = 2^e f, f in [sqrt(1/2), sqrt(2)); log f = 2 atanh(t), t = (f-1)/(f+1),
// |t| <= 0.1716: the odd series to t^25 is below 1e-20 relative.
SY_HD double sy_log(double x) {
    const uint64_t b = sy_double_as_u64(x);
    int e = (int)((b >> 52) & 0x7ff) - 1023;
    double f = sy_u64_as_double((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull);  // [1, 2)
    if (f > 1.4142135623730951) {
        f = SY_MUL(f, 0.5);
        e += 1;
    }
    const double t = SY_DIV(SY_SUB(f, 1.0), SY_ADD(f, 1.0));
    const double t2 = SY_MUL(t, t);
    // atanh(t)/t = sum t^(2k) / (2k+1), k = 0..12, Horner from the top
    double p = 1.0 / 25.0;
    p = SY_FMA(p, t2, 1.0 / 23.0);
    p = SY_FMA(p, t2, 1.0 / 21.0);
    p = SY_FMA(p, t2, 1.0 / 19.0);
    p = SY_FMA(p, t2, 1.0 / 17.0);
    p = SY_FMA(p, t2, 1.0 / 15.0);
    p = SY_FMA(p, t2, 1.0 / 13.0);
    p = SY_FMA(p, t2, 1.0 / 11.0);
    p = SY_FMA(p, t2, 1.0 / 9.0);
    p = SY_FMA(p, t2, 1.0 / 7.0);
    p = SY_FMA(p, t2, 1.0 / 5.0);
    p = SY_FMA(p, t2, 1.0 / 3.0);
    // log f = 2t + 2t^3 p'  with p' = (p - 1)/t2 folded: 2t * p
    const double tp = SY_MUL(SY_MUL(t, t2), p);  // t^3 * (1/3 + ...)
    const double lf = SY_MUL(2.0, SY_ADD(t, tp));
    const double LN2_HI = 6.93147180369123816490e-01;  // high 32 bits of ln 2
    const double LN2_LO = 1.90821492927058770002e-10;
    const double de = (double)e;
    return SY_ADD(SY_MUL(de, LN2_HI), SY_FMA(de, LN2_LO, lf));
}

// sin and cos of (pi/2) r for r in [0, 1/2]: Taylor series to x^21 / x^20.
SY_HD void sy_sincos_quarter(double r, double* s, double* c) {
    const double PIO2_HI = 1.57079632679489655800e+00;
    const double PIO2_LO = 6.12323399573676603587e-17;
    const double x = SY_FMA(r, PIO2_HI, SY_MUL(r, PIO2_LO));
    const double x2 = SY_MUL(x, x);
    double ps = -1.0 / 51090942171709440000.0;  // -1/21!
    ps = SY_FMA(ps, x2, 1.0 / 121645100408832000.0);  // 1/19!
    ps = SY_FMA(ps, x2, -1.0 / 355687428096000.0);    // -1/17!
    ps = SY_FMA(ps, x2, 1.0 / 1307674368000.0);       // 1/15!
    ps = SY_FMA(ps, x2, -1.0 / 6227020800.0);         // -1/13!
    ps = SY_FMA(ps, x2, 1.0 / 39916800.0);            // 1/11!
    ps = SY_FMA(ps, x2, -1.0 / 362880.0);             // -1/9!
    ps = SY_FMA(ps, x2, 1.0 / 5040.0);                // 1/7!
    ps = SY_FMA(ps, x2, -1.0 / 120.0);                // -1/5!
    ps = SY_FMA(ps, x2, 1.0 / 6.0);                   // 1/3!  (sign folded below)
    // sin x = x - x^3 (1/3! - x^2/5! + ...)
    *s = SY_SUB(x, SY_MUL(SY_MUL(x, x2), ps));
    double pc = 1.0 / 2432902008176640000.0;          // 1/20!
    pc = SY_FMA(pc, x2, -1.0 / 6402373705728000.0);   // -1/18!
    pc = SY_FMA(pc, x2, 1.0 / 20922789888000.0);      // 1/16!
    pc = SY_FMA(pc, x2, -1.0 / 87178291200.0);        // -1/14!
    pc = SY_FMA(pc, x2, 1.0 / 479001600.0);           // 1/12!
    pc = SY_FMA(pc, x2, -1.0 / 3628800.0);            // -1/10!
    pc = SY_FMA(pc, x2, 1.0 / 40320.0);               // 1/8!
    pc = SY_FMA(pc, x2, -1.0 / 720.0);                // -1/6!
    pc = SY_FMA(pc, x2, 1.0 / 24.0);                  // 1/4!
    pc = SY_FMA(pc, x2, -0.5);                        // -1/2!
    *c = SY_FMA(x2, pc, 1.0);
}

// The Gaussian pair number `pair` of stream `stream` under `seed`.
SY_HD void sy_gauss_pair(uint64_t seed, uint32_t stream, uint64_t pair, double* z0, double* z1) {
    uint32_t c[4] = {(uint32_t)pair, (uint32_t)(pair >> 32), stream, 0x5eed5eedu};
    sy_philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t x1 = ((uint64_t)c[0] << 32) | c[1];
    const uint64_t x2 = ((uint64_t)c[2] << 32) | c[3];
    const double u1 = SY_MUL((double)((x1 >> 11) + 1), 1.1102230246251565e-16);  // (0, 1]
    const uint64_t k = x2 >> 11;                                                    // u2 = k 2^-53
    // angle 2 pi u2 = (pi/2) (q + r), q = quadrant, r in [0, 1): exact split of 4 u2
    const uint32_t q = (uint32_t)(k >> 51);
    double r = SY_MUL((double)(k & ((1ull << 51) - 1)), 4.440892098500626e-16);  // 2^-51
    int swap = 0;
    if (r > 0.5) {
        r = SY_SUB(1.0, r);
        swap = 1;
    }
    double s, co;
    sy_sincos_quarter(r, &s, &co);
    if (swap) {
        const double t = s;
        s = co;
        co = t;
    }
    double sn, cs;
    switch (q) {
        case 0: sn = s; cs = co; break;
        case 1: sn = co; cs = -s; break;
        case 2: sn = -s; cs = -co; break;
        default: sn = -co; cs = s; break;
    }
    const double rad = SY_SQRT(SY_MUL(-2.0, sy_log(u1)));
    *z0 = SY_MUL(rad, cs);
    *z1 = SY_MUL(rad, sn);
}

// Element e of a stream: the pair e/2, cos half for even e, sin half for odd.
SY_HD double sy_gauss(uint64_t seed, uint32_t stream, uint64_t e) {
    double z0, z1;
    sy_gauss_pair(seed, stream, e >> 1, &z0, &z1);
    return (e & 1) ? z1 : z0;
}

// Quantised Gaussian: round(g 2^10) clamped to +-16383, times 2^-10 (exact).
SY_HD double sy_quantise_x(double g) {
    double a = SY_RINT(SY_MUL(g, 1024.0));
    if (a > SY_XMAX) a = SY_XMAX;
    if (a < -SY_XMAX) a = -SY_XMAX;
    return SY_MUL(a, 0.0009765625);
}
