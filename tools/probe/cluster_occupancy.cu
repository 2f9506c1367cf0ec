#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int *x) { extern __shared__ int s[]; if (threadIdx.x == 0 && x) x[blockIdx.x] = s[0]; }
int main() {
  for (int cs : {2, 4, 7, 8}) for (int smem_kb : {224, 112, 100}) for (int tpb : {512, 256}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(tpb); cfg.dynamicSmemBytes = smem_kb * 1024;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %d smem %d KB tpb %d: max active clusters %d (%d CTAs) %s\n", cs, smem_kb, tpb, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
