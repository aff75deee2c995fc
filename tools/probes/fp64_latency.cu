// Probe: dependent-chain latency of FP64 ops on sm_100a (one warp, clock64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double a, double b, int iters) {
    double x = threadIdx.x * 1e-3 + 1.0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    double y = x;
    for (int i = 0; i < iters; ++i) y = y * a;
    long long t2 = clock64();
    double z = y + 1.0;
    for (int i = 0; i < iters; ++i) z = sqrt(z);
    long long t3 = clock64();
    double w = z + 2.0;
    for (int i = 0; i < iters; ++i) w = 1.0 / w + 1.0;
    long long t4 = clock64();
    double v = w;
    for (int i = 0; i < iters; ++i) v = (double)rsqrtf((float)v) + 0.5;
    long long t5 = clock64();
    float f = (float)v;
    for (int i = 0; i < iters; ++i) f = fmaf(f, 1.0001f, 1e-3f);
    long long t6 = clock64();
    out[threadIdx.x] = x + y + z + w + v + f;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
    }
}

__global__ void barlat(long long* cyc, int iters) {
    __shared__ double s[1024];
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { s[threadIdx.x] = i; __syncthreads(); }
    long long t1 = clock64();
    double acc = 0;
    for (int i = 0; i < iters; ++i) { acc += s[(threadIdx.x + i) & 1023]; s[threadIdx.x] = acc; __syncthreads(); }
    long long t2 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}

int main() {
    double* d; long long* c; cudaMalloc(&d, 8 * 1024); cudaMalloc(&c, 64);
    long long h[8];
    const int it = 4096;
    lat<<<1, 32>>>(d, c, 1.0000001, 1e-9, it);
    cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: DFMA %.1f DMUL %.1f sqrt(f64) %.1f rcp(f64)+add %.1f rsqrtf-cvt+add %.1f FFMA %.1f\n",
           h[0] / (double)it, h[1] / (double)it, h[2] / (double)it, h[3] / (double)it, h[4] / (double)it, h[5] / (double)it);
    for (int t : {256, 384, 1024}) {
        barlat<<<1, t>>>(c, it);
        cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
        printf("threads %d: __syncthreads+STS %.1f cyc, LDS+DADD+STS+bar %.1f cyc\n", t, h[0] / (double)it, h[1] / (double)it);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
