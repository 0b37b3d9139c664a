// How many clusters of 2 / 4 / 8 / 16 CTAs (one CTA per SM: 200 KB of shared
// memory each) can be co-resident on this GPU (cudaOccupancyMaxActiveClusters).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_probe profiles/cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe_kernel(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"sms\": %d", sms);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe_kernel, &cfg);
    printf(", \"cluster_%d\": %d", cs, e == cudaSuccess ? n : -1);
  }
  printf("}\n");
  return 0;
}
