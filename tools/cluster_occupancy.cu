// How many 2-CTA clusters of a one-CTA-per-SM kernel fit on this GPU at once
// (cudaOccupancyMaxActiveClusters), for the smem sizes of the step kernel
// and the MoE GEMM. nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/co tools/cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dummy(int* p) {
  extern __shared__ int s[];
  if (p) p[threadIdx.x] = s[threadIdx.x];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smems[] = {200 * 1024, 227 * 1024};
  for (int cl : {1, 2, 4}) {
    for (int smem : smems) {
      cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(sms / cl * cl);
      cfg.blockDim = dim3(384);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cl;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = -1;
      const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
      std::printf("SMs %d, cluster %d, smem %d KB: max active clusters %d (%d CTAs) %s\n", sms, cl, smem / 1024, n,
                  n * cl, cudaGetErrorString(e));
    }
  }
  return 0;
}
