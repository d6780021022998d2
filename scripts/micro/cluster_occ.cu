// How many clusters of size 2/4/8 with one 224 KiB-smem CTA per SM can be co-resident on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int *p) { extern __shared__ int s[]; if (p) p[blockIdx.x] = s[threadIdx.x]; }
int main() {
    int smem = 224 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(148 * 4); cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = smem;
        cfg.attrs = attr; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cluster %2d: max active clusters %d -> %d SMs (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
    }
    return 0;
}
