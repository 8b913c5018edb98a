// Probe: how many thread-block clusters of a given size can be co-resident on this GPU
// (cudaOccupancyMaxActiveClusters), for the projection kernel's launch shape.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(double* p) { extern __shared__ double s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int cs : {2, 4, 8, 12, 16}) {
    for (int nt : {256, 512, 1024}) {
      for (int smem : {0, 65536, 131072}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 8, 1, 1);
        cfg.blockDim = dim3(nt, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = cs; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
        cfg.attrs = &attr; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        printf("cluster %2d threads %4d smem %6d -> max active clusters %d (%s)\n", cs, nt, smem, n,
               cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
