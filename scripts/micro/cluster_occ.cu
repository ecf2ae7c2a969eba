// Dev probe: co-resident clusters per cluster size / dynamic shared memory on this GPU
// (cudaOccupancyMaxActiveClusters), for planning the narrow engine's cluster shapes.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(float* p) { extern __shared__ float s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int kbs[] = {48, 100, 120, 150, 200, 227};
  printf("smemKB:");
  for (int kb : kbs) printf(" %5d", kb);
  printf("\n");
  for (int nc = 1; nc <= 16; ++nc) {
    printf("nc=%2d :", nc);
    for (int kb : kbs) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nc); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = kb * 1024;
      cudaLaunchAttribute a; a.id = cudaLaunchAttributeClusterDimension; a.val.clusterDim.x = nc; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
      cfg.attrs = &a; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)dummy, &cfg);
      printf(" %5d", e == cudaSuccess ? n : -1);
    }
    printf("\n");
  }
  return 0;
}
