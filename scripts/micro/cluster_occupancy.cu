// How many clusters of 2 / 4 / 8 CTAs (one CTA per SM, ~199 KB SMEM each) can
// be co-resident on this GPU (cudaOccupancyMaxActiveClusters)?  Analysis only.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { if (p) p[0] = 1; }
int main() {
  const int smem = 198656;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = smem; cfg.attrs = attr; cfg.numAttrs = 1;
    cfg.gridDim = dim3(sms);
    int nc = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
    printf("cluster %2d: max active clusters %d -> %d SMs of %d (%s)\n", cs, nc, nc * cs, sms, cudaGetErrorString(e));
  }
  return 0;
}
