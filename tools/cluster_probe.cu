// Max co-resident clusters of k_dense_run's shape (352 threads, 225 KB smem) per cluster
// size: whether 4-CTA clusters (two tcgen05 pairs) can cover all 148 SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/_cluster_probe tools/cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dummy(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
    const int smem = 224 * 1024 + 1024 + 256;
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148 / cs * cs);
        cfg.blockDim = dim3(352);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
        printf("cluster %d: max active clusters %d (%d SMs) %s\n", cs, n, n * cs,
               cudaGetErrorString(e));
    }
    return 0;
}
