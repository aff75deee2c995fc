// H2D bandwidth of a column-major pinned matrix: one contiguous copy vs row
// chunks as cudaMemcpy2DAsync (n segments of rows*8 bytes, pitch m*8).
//   nvcc -O2 -o tools/probes/h2d2d tools/probes/h2d2d.cu && tools/probes/h2d2d 200000 1024 32768
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

int main(int argc, char** argv) {
    const size_t m = argc > 1 ? atol(argv[1]) : 200000, n = argc > 2 ? atol(argv[2]) : 1024;
    const size_t rows = argc > 3 ? atol(argv[3]) : 32768;
    double *h, *d;
    cudaMallocHost(&h, m * n * 8);
    cudaMalloc(&d, m * n * 8);
    for (size_t i = 0; i < m * n; i += 512) h[i] = 1.0;
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a, s);
        cudaMemcpyAsync(d, h, m * n * 8, cudaMemcpyHostToDevice, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("contiguous: %.2f ms = %.1f GB/s\n", ms, m * n * 8 / ms / 1e6);
        cudaEventRecord(a, s);
        auto t0 = std::chrono::steady_clock::now();
        for (size_t r0 = 0; r0 < m; r0 += rows) {
            const size_t mk = r0 + rows < m ? rows : m - r0;
            cudaMemcpy2DAsync(d + r0, m * 8, h + r0, m * 8, mk * 8, n, cudaMemcpyHostToDevice, s);
        }
        const double host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        printf("  host time to enqueue the 2-D copies: %.2f ms\n", host_ms);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("2-D row chunks of %zu: %.2f ms = %.1f GB/s (%s)\n", rows, ms, m * n * 8 / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
