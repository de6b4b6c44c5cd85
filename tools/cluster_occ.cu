// Max co-resident clusters per cluster size at ~200 KB shared memory per CTA (dev tool).
#include <cstdio>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 3, 4, 5, 6, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = cs; la[0].val.clusterDim.y = 1; la[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = 200 * 1024;
    cfg.attrs = la; cfg.numAttrs = 1;
    int v = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&v, k, &cfg);
    printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", cs, v, v * cs, cudaGetErrorString(e));
  }
  return 0;
}
