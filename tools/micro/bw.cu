// Microbenchmark (dev tool, not product): read bandwidth of (a) LDG.128 grid-stride loop,
// (b) cp.async.bulk ring into smem with N stages of S KB, over a 512 MB buffer.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned s_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void ldg_kernel(const float4* __restrict__ x, size_t n4, float* out) {
  float acc = 0.f;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 8
  for (; i < n4; i += stride) { float4 v = __ldcs(x + i); acc += v.x + v.y + v.z + v.w; }
  if (acc == 12345.f) out[0] = acc;
}
template <int NS>
__global__ void bulk_kernel(const float* __restrict__ x, size_t nfl, int stage_fl, float* out) {
  extern __shared__ __align__(128) float buf[];
  __shared__ unsigned long long bar[NS];
  size_t per = (nfl / gridDim.x) & ~(size_t)3;
  const float* base = x + per * blockIdx.x;
  int nst = (int)(per / stage_fl);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int s) {
    int slot = s % NS;
    unsigned bytes = stage_fl * 4;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&bar[slot])), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(s_u32(buf + (size_t)slot * stage_fl)), "l"(base + (size_t)s * stage_fl), "r"(bytes), "r"(s_u32(&bar[slot])) : "memory");
  };
  if (threadIdx.x == 0) for (int s = 0; s < NS && s < nst; ++s) issue(s);
  float acc = 0.f;
  for (int s = 0; s < nst; ++s) {
    int slot = s % NS;
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(s_u32(&bar[slot])), "r"((unsigned)(s / NS) & 1u) : "memory");
    const float4* b4 = reinterpret_cast<const float4*>(buf + (size_t)slot * stage_fl);
    for (int i = threadIdx.x; i < stage_fl / 4; i += blockDim.x) { float4 v = b4[i]; acc += v.x + v.y + v.z + v.w; }
    __syncthreads();
    if (threadIdx.x == 0 && s + NS < nst) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(s + NS); }
  }
  if (acc == 12345.f) out[0] = acc;
}
int main() {
  size_t bytes = 512ull << 20; float* x; float* out; cudaMalloc(&x, bytes); cudaMalloc(&out, 4);
  cudaMemset(x, 0, bytes);
  char* fl; cudaMalloc(&fl, 256ull << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto f) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(fl, it, 256ull << 20);
      cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("%-40s %8.1f us  %7.1f GB/s  err=%s\n", name, best * 1e3, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  for (int bpsm : {1, 2, 4, 8}) {
    char nm[64]; snprintf(nm, 64, "ldg128 blocks=148x%d thr=512", bpsm);
    run(nm, [&] { ldg_kernel<<<148 * bpsm, 512>>>((const float4*)x, bytes / 16, out); });
  }
  for (int skb : {16, 32, 48}) for (int ns : {2, 4, 6}) {
    int sfl = skb * 256; size_t smem = (size_t)ns * sfl * 4; if (smem > 220 * 1024) continue;
    char nm[64]; snprintf(nm, 64, "bulk ns=%d stage=%dKB grid=148", ns, skb);
    if (ns == 2) { cudaFuncSetAttribute(bulk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); run(nm, [&] { bulk_kernel<2><<<148, 512, smem>>>(x, bytes / 4, sfl, out); }); }
    if (ns == 4) { cudaFuncSetAttribute(bulk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); run(nm, [&] { bulk_kernel<4><<<148, 512, smem>>>(x, bytes / 4, sfl, out); }); }
    if (ns == 6) { cudaFuncSetAttribute(bulk_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); run(nm, [&] { bulk_kernel<6><<<148, 512, smem>>>(x, bytes / 4, sfl, out); }); }
  }
  // 2 CTAs per SM
  { int ns = 4, sfl = 16 * 256; size_t smem = (size_t)ns * sfl * 4; cudaFuncSetAttribute(bulk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    run("bulk ns=4 stage=16KB grid=296", [&] { bulk_kernel<4><<<296, 256, smem>>>(x, bytes / 4, sfl, out); }); }
  return 0;
}
