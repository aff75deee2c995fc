// Probe: latency of one Jacobi rotation-parameter evaluation (dependent chain).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_nr(double x) {
    double y = static_cast<double>(rsqrtf(static_cast<float>(x)));
    const double h = 0.5 * x;
    y = y * fma(-h * y, y, 1.5);
    y = y * fma(-h * y, y, 1.5);
    return y;
}
__device__ __forceinline__ void rot_fast(double app, double aqq, double apq, double& c, double& s) {
    double d = aqq - app, e = 2.0 * apq;
    const double big = fmax(fabs(d), fabs(e));
    if (!(big < 0x1p60 && big > 0x1p-60)) {
        const double scale = scalbn(1.0, -ilogb(big));
        d *= scale;
        e *= scale;
    }
    const double r2 = fma(d, d, e * e);
    const double D = fabs(d) + r2 * rsqrt_nr(r2);
    const double inv = rsqrt_nr(fma(D, D, e * e));
    c = D * inv;
    s = (d > 0.0 ? e : (d < 0.0 ? -e : fabs(e))) * inv;
}
__device__ __forceinline__ void rot_nocheck(double app, double aqq, double apq, double& c, double& s) {
    double d = aqq - app, e = 2.0 * apq;
    const double r2 = fma(d, d, e * e);
    const double D = fabs(d) + r2 * rsqrt_nr(r2);
    const double inv = rsqrt_nr(fma(D, D, e * e));
    c = D * inv;
    s = copysign(1.0, d) * e * inv;
}
__device__ __forceinline__ void rot_ref(double app, double aqq, double apq, double& c, double& s) {
    const double tau = (aqq - app) / (2.0 * apq);
    double t;
    if (tau >= 0.0) t = 1.0 / (tau + sqrt(1.0 + tau * tau));
    else t = -1.0 / (-tau + sqrt(1.0 + tau * tau));
    c = 1.0 / sqrt(1.0 + t * t);
    s = t * c;
}
__device__ __forceinline__ void rot_rsq(double app, double aqq, double apq, double& c, double& s) {
    double d = aqq - app, e = 2.0 * apq;
    const double r2 = fma(d, d, e * e);
    const double D = fabs(d) + r2 * rsqrt(r2);
    const double inv = rsqrt(fma(D, D, e * e));
    c = D * inv;
    s = copysign(1.0, d) * e * inv;
}

template <int V>
__global__ void k(double* out, long long* cyc, int iters) {
    double a = 1.0 + threadIdx.x, b = 2.5, x = 0.3;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double c, s;
        if (V == 0) rot_fast(a, b, x, c, s);
        if (V == 1) rot_nocheck(a, b, x, c, s);
        if (V == 2) rot_ref(a, b, x, c, s);
        if (V == 3) rot_rsq(a, b, x, c, s);
        x = 0.25 * s + 0.1;  // dependent chain
        a = c;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x + a;
    if (threadIdx.x == 0) cyc[V] = t1 - t0;
}

int main() {
    double* d; long long* c; cudaMalloc(&d, 8 * 64); cudaMalloc(&c, 64);
    const int it = 1000;
    k<0><<<1, 32>>>(d, c, it); k<1><<<1, 32>>>(d, c, it); k<2><<<1, 32>>>(d, c, it); k<3><<<1, 32>>>(d, c, it);
    long long h[4];
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("rotation latency (cycles): fast %.0f  nocheck %.0f  reference %.0f  cuda-rsqrt %.0f\n", h[0] / (double)it,
           h[1] / (double)it, h[2] / (double)it, h[3] / (double)it);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
