// Read-bandwidth ceiling probe (B200): (a) plain LDG.128 streaming with 8 loads in flight per
// thread, (b) a TMA bulk ring (2 x 96 KB per CTA, one CTA per SM) whose consumer does no work.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_bw read_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ldg_kernel(const float4* __restrict__ x, size_t n4, float* out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n4; i += stride) { float4 v = __ldcs(x + i); acc += v.x + v.y + v.z + v.w; }
  if (acc == 123.456f) out[0] = acc;
}

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void tma_kernel(const float* __restrict__ x, size_t nbytes, unsigned stage, int ns, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long bar[8];
  const size_t per = (nbytes / gridDim.x) / stage * stage;
  const char* base = reinterpret_cast<const char*>(x) + per * blockIdx.x;
  const int nst = (int)(per / stage);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int s) {
    const int slot = s % ns;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[slot])), "r"(stage) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su(sm + (size_t)slot * stage)),
                 "l"(base + (size_t)s * stage), "r"(stage), "r"(su(&bar[slot]))
                 : "memory");
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < ns && s < nst; ++s) issue(s);
  float acc = 0.f;
  for (int s = 0; s < nst; ++s) {
    const int slot = s % ns;
    const unsigned par = (unsigned)(s / ns) & 1u;
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                     su(&bar[slot])), "r"(par) : "memory");
    acc += reinterpret_cast<const float*>(sm + (size_t)slot * stage)[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && s + ns < nst) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(s + ns);
    }
  }
  if (acc == 123.456f) out[0] = acc;
}

int main() {
  const size_t nbytes = (size_t)40 << 30;
  float* x; float* out;
  if (cudaMalloc(&x, nbytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&out, 4);
  cudaMemset(x, 0, nbytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bps : {4, 8}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      ldg_kernel<<<148 * bps, 256>>>(reinterpret_cast<const float4*>(x), nbytes / 16, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("ldg blocks/SM %d: %.1f GB/s\n", bps, nbytes / ms / 1e6);
    }
  }
  struct { unsigned stage; int ns; } cfgs[] = {{96 << 10, 2}, {64 << 10, 3}, {48 << 10, 4}, {32 << 10, 6}, {24 << 10, 8}, {100 << 10, 2}};
  for (auto c : cfgs) {
    const size_t smem = (size_t)c.stage * c.ns;
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      tma_kernel<<<148, 256, smem>>>(x, nbytes, c.stage, c.ns, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("tma stage %u KB x %d: %.1f GB/s (%s)\n", c.stage >> 10, c.ns, nbytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
