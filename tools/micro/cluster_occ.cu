// Microbenchmark (dev tool): co-resident clusters and SM placement for cluster sizes / smem /
// block sizes of interest (which SMs the CTAs of 8 clusters land on).
#include <cstdio>
#include <set>
#include <cuda_runtime.h>
__global__ void k(int* smid) {
  unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) smid[blockIdx.x] = (int)s;
  long long t = clock64(); while (clock64() - t < 2000000) {}
}
int main() {
  int* d; cudaMalloc(&d, 4096 * 4);
  for (int threads : {512}) for (int smemkb : {200}) for (int cs : {9, 10, 11, 12, 13, 14, 15, 16}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smemkb * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(cs * 8); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smemkb * 1024;
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int act = 0; cudaOccupancyMaxActiveClusters(&act, k, &cfg);
    cudaLaunchKernelEx(&cfg, k, d); cudaDeviceSynchronize();
    int h[4096]; cudaMemcpy(h, d, cs * 8 * 4, cudaMemcpyDeviceToHost);
    std::set<int> sms(h, h + cs * 8);
    printf("threads=%d smem=%dKB CS=%2d: act=%3d, 8 clusters on %zu distinct SMs (%d CTAs) %s\n", threads, smemkb, cs, act,
           sms.size(), cs * 8, cudaGetErrorString(cudaGetLastError()));
  }
}
