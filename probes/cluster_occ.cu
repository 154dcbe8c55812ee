// Probe: how many thread-block clusters of size 8 / 16 (non-portable) with the
// attention kernel's footprint (256 threads, ~144 KB dynamic smem) can be resident.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(1, 1, 1) dummy_fixed() {}
__global__ void k(int* out) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0) sm[0] = 1;
  if (out && threadIdx.x == 0) out[blockIdx.x] = sm[0];
}
int main() {
  int smem = 144 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 8, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %d (%s) -> %d CTAs\n", cs, n, cudaGetErrorString(e), n * cs);
    for (int sm2 : {80 * 1024, 40 * 1024}) {
      cfg.dynamicSmemBytes = sm2;
      e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("    smem %d KB: %d clusters (%d CTAs)\n", sm2 / 1024, n, n * cs);
      cfg.dynamicSmemBytes = smem;
    }
  }
  return 0;
}
