// Probe: accuracy and latency of the speculative-seed rotation (rotation_fast in
// csrc/jacobi.cu) against the rsqrt()-based one, over random (app, aqq, apq).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

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
__device__ __forceinline__ void rot_fast(double app, double aqq, double apq, double& c, double& s) {
    const double d = aqq - app, e = 2.0 * apq, e2 = e * e, ad = fabs(d);
    const double r2 = fma(d, d, e2);
    const double y0 = rsqrt_seed(r2);
    const double Dt = ad + r2 * y0;
    const double z0 = rsqrt_seed(fma(Dt, Dt, e2));
    const double D = ad + r2 * rsqrt_refine(r2, y0);
    const double inv = rsqrt_refine(fma(D, D, e2), z0);
    c = D * inv;
    s = (d > 0.0 ? e : (d < 0.0 ? -e : fabs(e))) * inv;
}
__device__ __forceinline__ void rot_rsq(double app, double aqq, double apq, double& c, double& s) {
    const double d = aqq - app, e = 2.0 * apq;
    const double r2 = fma(d, d, e * e);
    const double D = fabs(d) + r2 * rsqrt(r2);
    const double inv = rsqrt(fma(D, D, e * e));
    c = D * inv;
    s = (d > 0.0 ? e : (d < 0.0 ? -e : fabs(e))) * inv;
}
__device__ unsigned long long rng(unsigned long long& st) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    return st;
}
__global__ void acc(double* out, int iters) {
    unsigned long long st = 0x9E3779B97F4A7C15ull * (threadIdx.x + 1 + 1024 * blockIdx.x);
    double worst_cs = 0, worst_norm = 0, worst_seed = 0, worst_ann = 0;
    for (int i = 0; i < iters; ++i) {
        auto u = [&]() { return (rng(st) >> 11) * (1.0 / 9007199254740992.0); };
        const double sc = exp2(floor(60.0 * u() - 30.0));
        const double app = sc * (2 * u() - 1), aqq = sc * (2 * u() - 1) * exp2(floor(-20 * u()));
        const double apq = sc * (2 * u() - 1) * exp2(floor(-40 * u()));
        double c0, s0, c1, s1;
        rot_rsq(app, aqq, apq, c0, s0);
        rot_fast(app, aqq, apq, c1, s1);
        worst_cs = fmax(worst_cs, fmax(fabs(c1 - c0), fabs(s1 - s0) / fmax(fabs(s0), 1e-300)));
        worst_norm = fmax(worst_norm, fabs(fma(c1, c1, s1 * s1) - 1.0));
        const double x = fabs(app) + 1e-3;
        worst_seed = fmax(worst_seed, fabs(rsqrt_seed(x) * sqrt(x) - 1.0));
        // residual coupling after the rotation relative to |apq|
        const double r = (c1 * c1 - s1 * s1) * apq + c1 * s1 * (app - aqq);
        worst_ann = fmax(worst_ann, fabs(r) / (fabs(apq) + 1e-300) * fmin(1.0, fabs(apq) / fmax(fabs(app - aqq), 1e-300)));
    }
    atomicMax(reinterpret_cast<unsigned long long*>(out), __double_as_longlong(worst_cs));
    atomicMax(reinterpret_cast<unsigned long long*>(out + 1), __double_as_longlong(worst_norm));
    atomicMax(reinterpret_cast<unsigned long long*>(out + 2), __double_as_longlong(worst_seed));
    atomicMax(reinterpret_cast<unsigned long long*>(out + 3), __double_as_longlong(worst_ann));
}
template <int V>
__global__ void lat(double* out, long long* cyc, int iters) {
    double a = 1.0 + threadIdx.x, b = 2.5, x = 0.3;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double c, s;
        if (V == 0) rot_fast(a, b, x, c, s); else rot_rsq(a, b, x, c, s);
        a = fma(c, 1e-9, a);
        x = fma(s, 1e-9, x);
    }
    cyc[0] = (clock64() - t0) / iters;
    out[threadIdx.x] = a + x;
}
int main() {
    double* d; long long* c;
    cudaMalloc(&d, 64 * sizeof(double)); cudaMalloc(&c, 8);
    cudaMemset(d, 0, 64 * sizeof(double));
    acc<<<64, 256>>>(d, 20000);
    double h[4]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("max |dc|, rel ds vs rsqrt version: %.3e\nmax |c^2+s^2-1|: %.3e\nmax rel error of the hardware seed: %.3e (2^%.1f)\nannihilation residual (scaled): %.3e\n",
           h[0], h[1], h[2], log2(h[2]), h[3]);
    long long hc;
    lat<0><<<1, 32>>>(d, c, 2000); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost); printf("rotation_fast: %lld cycles\n", hc);
    lat<1><<<1, 32>>>(d, c, 2000); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost); printf("rotation (rsqrt): %lld cycles\n", hc);
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
