// Microbenchmark (dev tool): the ALS pass inner product pattern acc[4][12] += y[c] * w[f]
// with scalar FFMA vs packed fma.rn.f32x2 (FFMA2), operands from shared memory as in the pass.
#include <cstdio>
#include <cuda_runtime.h>

template <bool PACKED>
__global__ void __launch_bounds__(512, 1) k_pat(const float* __restrict__ g, float* out, int rows) {
  __shared__ __align__(16) float sy[128 * 4 * 8];
  __shared__ __align__(16) float sw[128 * 12];
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) sy[i] = g[i & 1023] * 0.5f;
  for (int i = threadIdx.x; i < 128 * 12; i += blockDim.x) sw[i] = g[i & 1023] * 0.25f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float acc[4][12];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int f = 0; f < 12; ++f) acc[c][f] = 0.f;
  for (int it = 0; it < rows; ++it) {
    const int row = it & 31;
    const float4 y = *reinterpret_cast<const float4*>(sy + row * 128 + 4 * lane);
    float w[12];
#pragma unroll
    for (int f4 = 0; f4 < 3; ++f4) {
      const float4 v = reinterpret_cast<const float4*>(sw + row * 12)[f4];
      w[4 * f4] = v.x; w[4 * f4 + 1] = v.y; w[4 * f4 + 2] = v.z; w[4 * f4 + 3] = v.w;
    }
    if (!PACKED) {
#pragma unroll
      for (int f = 0; f < 12; ++f) {
        acc[0][f] = fmaf(y.x, w[f], acc[0][f]);
        acc[1][f] = fmaf(y.y, w[f], acc[1][f]);
        acc[2][f] = fmaf(y.z, w[f], acc[2][f]);
        acc[3][f] = fmaf(y.w, w[f], acc[3][f]);
      }
    } else {
      // pairs over f: acc[c][f..f+1] += y.c * w[f..f+1]
      const float yc[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int f = 0; f < 12; f += 2) {
          unsigned long long a, b, d;
          asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(yc[c]), "f"(yc[c]));
          asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(w[f]), "f"(w[f + 1]));
          asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(acc[c][f]), "f"(acc[c][f + 1]));
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
          asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[c][f]), "=f"(acc[c][f + 1]) : "l"(d));
        }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int f = 0; f < 12; ++f) s += acc[c][f];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float *g, *out;
  cudaMalloc(&g, 4096 * 4);
  cudaMemset(g, 0, 4096 * 4);
  cudaMalloc(&out, 148 * 512 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int rows = 20000;
  for (int warps : {4, 8, 12, 16}) {
    for (int packed = 0; packed < 2; ++packed) {
      float ms;
      auto k = packed ? k_pat<true> : k_pat<false>;
      k<<<148, warps * 32>>>(g, out, 100);
      cudaEventRecord(e0); k<<<148, warps * 32>>>(g, out, rows); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double fma = 148.0 * warps * 32 * rows * 48;
      printf("%s warps/SM=%2d: %.0f FMA/clk/SM, %.2f cycles per row per warp-slot\n", packed ? "f32x2" : "ffma ",
             warps, fma / (ms * 1e-3) / 148 / 1.965e9, (ms * 1e-3 * 1.965e9) / rows / (warps / 4.0));
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
