// Probe: how many clusters of size CS can be co-resident (one CTA per SM,
// ~145 KB dynamic shared memory, 288 threads), i.e. whether a grid of
// floor(148 / CS) clusters runs in a single wave.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dummy(int* p) {
    extern __shared__ int s[];
    if (p) p[0] = s[threadIdx.x];
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int smem_kb : {145, 200}) {
        for (int cs : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(sms / cs * cs);
            cfg.blockDim = dim3(288);
            cfg.dynamicSmemBytes = smem_kb * 1024;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cs;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
            printf("smem %3d KB  cluster %2d: max active clusters %3d (= %3d CTAs of %d SMs) %s\n", smem_kb, cs,
                   n, n * cs, sms, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
