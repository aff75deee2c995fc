// Probe: cost of one "Cholesky-like" step (serial FP64 pivot chain by one
// thread + barrier + row scale + barrier + warp-per-column smem update +
// barrier) with 256 threads on a 64x65 shared-memory tile.
#include <cstdio>
#include <cuda_runtime.h>

template <int VARIANT>
__global__ void step_kernel(double* out, long long* cyc, int steps) {
    constexpr int LD = 65, BS = 64;
    __shared__ double S[BS * LD];
    __shared__ double dinv[BS];
    const int tid = threadIdx.x;
    for (int e = tid; e < BS * LD; e += blockDim.x) S[e] = 1.0 + (e % 7) * 1e-3 + (e % LD == e / LD ? 100.0 : 0.0);
    __syncthreads();
    long long t0 = clock64();
    for (int j = 0; j < steps; ++j) {
        if (tid == 0) {
            const double d = S[j + j * LD];
            const double r = (VARIANT & 1) ? d * 0.5 + 0.25 : sqrt(fmax(d, 0.0));
            S[j + j * LD] = r;
            dinv[j] = (VARIANT & 1) ? r : 1.0 / r;
        }
        __syncthreads();
        const double inv = dinv[j];
        for (int c = j + 1 + tid; c < BS; c += blockDim.x) S[j + c * LD] *= inv;
        __syncthreads();
        if (!(VARIANT & 2)) {
            const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
            for (int cc = j + 1 + warp; cc < BS; cc += nw) {
                const double sjc = S[j + cc * LD];
                for (int i = j + 1 + lane; i <= cc; i += 32) S[i + cc * LD] -= S[j + i * LD] * sjc;
            }
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[VARIANT] = (t1 - t0) / steps;
    out[tid] = S[tid];
}

int main() {
    double* d; long long* c; cudaMalloc(&d, 8 * 1024); cudaMalloc(&c, 64);
    step_kernel<0><<<1, 256>>>(d, c, 63);
    step_kernel<1><<<1, 256>>>(d, c, 63);
    step_kernel<2><<<1, 256>>>(d, c, 63);
    step_kernel<3><<<1, 256>>>(d, c, 63);
    long long h[4];
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("cycles/step: full %lld | no sqrt/div %lld | no update %lld | neither %lld\n", h[0], h[1], h[2], h[3]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
