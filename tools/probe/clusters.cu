#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(2, 1, 1) k2(int* p) { if (p) p[0] = 1; }
__global__ void __cluster_dims__(4, 1, 1) k4(int* p) { if (p) p[0] = 1; }
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int smem : {16 << 10, 64 << 10, 128 << 10, 200 << 10}) {
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
    int c2 = 0, c4 = 0;
    cudaOccupancyMaxActiveClusters(&c2, k2, &cfg);
    cudaOccupancyMaxActiveClusters(&c4, k4, &cfg);
    printf("sms %d smem %d KB: max active 2-CTA clusters %d (%d CTAs), 4-CTA %d (%d CTAs)\n", sms, smem >> 10, c2, 2 * c2, c4, 4 * c4);
  }
  return 0;
}
