// Probe: HBM read bandwidth of TMA slab streaming over a column-major
// m x n FP64 matrix, as a function of the box shape (rows x cols, 16 KB per
// box), the number of passes (pass 2 re-reads the slab, evict_last/first
// hints), and the slab -> CTA assignment. No arithmetic: isolates the
// access pattern of the Lanczos GEMV pair from its compute.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1906_12085_b200/csrc \
//        stream_tma.cu -o stream_tma -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "tma_util.h"

using namespace svdk;

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

namespace svdk {
CUtensorMap tensor_map_2d(const double* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box0,
                          uint32_t box1, CUtensorMapSwizzle swizzle) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    cuuint32_t box[2] = {box0, box1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                       es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", r);
        exit(1);
    }
    return m;
}
}  // namespace svdk

constexpr int NCW = 8;

// ASSIGN 0: slab s -> CTA s % grid (interleaved); 1: contiguous slab ranges per CTA;
// CS > 1: CS consecutive CTAs share a slab, each streaming n/CS of its columns
template <int R, int C, int PASSES, int ASSIGN, int CS = 1>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    stream_kernel(const __grid_constant__ CUtensorMap map, long long m, long long n, double* sink) {
    extern __shared__ uint8_t raw[];
    double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NCW * R * C);
    uint64_t* empty = full + NCW;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = (int)(n / C / CS);
    const int tcol0 = (int)(blockIdx.x % CS) * T;
    const long long nslabs = m / R;
    long long s_begin, s_end, s_step;
    if (ASSIGN == 0) {
        s_begin = blockIdx.x / CS; s_end = nslabs; s_step = gridDim.x / CS;
    } else {
        const long long per = (nslabs + gridDim.x - 1) / gridDim.x;
        s_begin = blockIdx.x * per; s_end = s_begin + per < nslabs ? s_begin + per : nslabs; s_step = 1;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < NCW; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NCW) {
        if (lane == 0) {
            const uint64_t keep = l2_policy_evict_last(), drop = l2_policy_evict_first();
            long long k = 0;
            for (long long sl = s_begin; sl < s_end; sl += s_step)
                for (int pass = 0; pass < PASSES; ++pass)
                    for (int t = 0; t < T; ++t, ++k) {
                        const int st = (int)(k % NCW);
                        const uint32_t use = (uint32_t)(k / NCW);
                        mbar_wait(&empty[st], (use & 1) ^ 1);
                        mbar_expect_tx(&full[st], R * C * 8);
                        tma_load_2d_hint(ring + st * R * C, &map, &full[st], (int)(sl * R), (tcol0 + t) * C,
                                         (PASSES == 1 || pass == 1) ? drop : keep);
                    }
        }
        return;
    }
    double acc = 0.0;
    uint32_t uses = 0;
    long long k0 = 0;
    for (long long sl = s_begin; sl < s_end; sl += s_step)
        for (int pass = 0; pass < PASSES; ++pass)
            for (int t = 0; t < T; ++t, ++k0) {
                if ((int)(k0 % NCW) != warp) continue;
                mbar_wait(&full[warp], uses & 1);
                acc += ring[warp * R * C + lane];
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[warp]);
                ++uses;
            }
    if (acc == 12345.0) sink[0] = acc;
}

// plain streaming read: thread-coalesced double2 over the whole matrix
__global__ void plain_read(const double2* a, long long count, double* sink) {
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        double2 v = __ldcs(a + i);
        acc += v.x + v.y;
    }
    if (acc == 12345.0) sink[0] = acc;
}

template <int R, int C, int PASSES, int ASSIGN, int CS = 1>
void run(const double* A, long long m, long long n, double* sink, int sms, const char* name) {
    CUtensorMap map = tensor_map_2d(A, m, n, m, R, C, CU_TENSOR_MAP_SWIZZLE_NONE);
    size_t smem = 128 + NCW * R * C * 8 + 2 * NCW * 8;
    cudaFuncSetAttribute(stream_kernel<R, C, PASSES, ASSIGN, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
        cudaEventRecord(e0);
        stream_kernel<R, C, PASSES, ASSIGN, CS><<<sms, (NCW + 1) * 32, smem>>>(map, m, n, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0 && ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("%-34s %8.3f ms  %7.0f GB/s (one read of A)  %s\n", name, best, m * n * 8.0 / best / 1e6,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main(int argc, char** argv) {
    long long m = argc > 1 ? atoll(argv[1]) : 500000;
    long long n = argc > 2 ? atoll(argv[2]) : 2048;
    m = m / 256 * 256;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *A, *sink;
    cudaMalloc(&A, m * n * 8);
    cudaMalloc(&sink, 64);
    cudaMemset(A, 0, m * n * 8);
    printf("m=%lld n=%lld (%.2f GB), %d SMs\n", m, n, m * n * 8e-9, sms);
    {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaEventRecord(e0);
            plain_read<<<sms * 4, 512>>>((const double2*)A, m * n / 2, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it > 0 && ms < best) best = ms;
        }
        printf("%-34s %8.3f ms  %7.0f GB/s\n", "plain double2 read", best, m * n * 8.0 / best / 1e6);
    }
    run<32, 64, 2, 0, 2>(A, m, n, sink, sms, "32x64 2pass split2 (L2 reuse)");
    run<32, 64, 2, 0, 4>(A, m, n, sink, sms, "32x64 2pass split4 (L2 reuse)");
    run<64, 32, 2, 0, 2>(A, m, n, sink, sms, "64x32 2pass split2 (L2 reuse)");
    run<64, 32, 2, 0, 4>(A, m, n, sink, sms, "64x32 2pass split4 (L2 reuse)");
    run<128, 16, 2, 0, 4>(A, m, n, sink, sms, "128x16 2pass split4 (L2 reuse)");
    run<32, 64, 1, 0>(A, m, n, sink, sms, "32x64 1pass interleaved");
    run<64, 32, 1, 0>(A, m, n, sink, sms, "64x32 1pass interleaved");
    run<128, 16, 1, 0>(A, m, n, sink, sms, "128x16 1pass interleaved");
    run<256, 8, 1, 0>(A, m, n, sink, sms, "256x8 1pass interleaved");
    run<32, 64, 1, 1>(A, m, n, sink, sms, "32x64 1pass contiguous");
    run<32, 64, 2, 0>(A, m, n, sink, sms, "32x64 2pass interleaved (L2 reuse)");
    run<32, 64, 2, 1>(A, m, n, sink, sms, "32x64 2pass contiguous (L2 reuse)");
    run<64, 32, 2, 0>(A, m, n, sink, sms, "64x32 2pass interleaved (L2 reuse)");
    run<16, 128, 1, 0>(A, m, n, sink, sms, "16x128 1pass interleaved");
    run<16, 128, 2, 0>(A, m, n, sink, sms, "16x128 2pass interleaved");
    return 0;
}
