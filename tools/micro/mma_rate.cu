// Microbenchmark (dev tool): issue rate of legacy warp MMA (mma.sync m16n8k8 tf32,
// m16n8k16 bf16) and of 3-register FFMA on one B200, all SMs busy.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tf32(float* out, int iters) {
  unsigned a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
  unsigned b[2] = {threadIdx.x * 3u, threadIdx.x * 5u};
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_bf16(float* out, int iters) {
  unsigned a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
  unsigned b[2] = {threadIdx.x * 3u, threadIdx.x * 5u};
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(float* out, int iters, float x, float y) {
  float c[32];
  for (int j = 0; j < 32; ++j) c[j] = threadIdx.x + j;
  float w = x * threadIdx.x;
  const float y2 = y + 1e-3f * threadIdx.x;   // per-thread register: 3-register FFMA form
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) c[j] = fmaf(c[j], w, y2);
    w += 1e-7f;
  }
  float s = 0;
  for (int j = 0; j < 32; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148;
  for (int warps : {4, 8, 16}) {
    const int blocks = sms * 2, th = 32 * warps, it = 4096;
    float ms;
    k_tf32<<<blocks, th>>>(out, 16);
    cudaEventRecord(e0); k_tf32<<<blocks, th>>>(out, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double macs = (double)blocks * warps * it * 8 * 16 * 8 * 8;
    printf("tf32 m16n8k8 warps/CTA=%d: %.1f TFLOP/s  (%.0f MAC/clk/SM @1.965GHz)\n", warps, 2 * macs / ms / 1e9,
           macs / (ms * 1e-3) / 148 / 1.965e9);
    k_bf16<<<blocks, th>>>(out, 16);
    cudaEventRecord(e0); k_bf16<<<blocks, th>>>(out, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    macs = (double)blocks * warps * it * 8 * 16 * 8 * 16;
    printf("bf16 m16n8k16 warps/CTA=%d: %.1f TFLOP/s  (%.0f MAC/clk/SM)\n", warps, 2 * macs / ms / 1e9,
           macs / (ms * 1e-3) / 148 / 1.965e9);
    k_ffma<<<blocks, th>>>(out, 16, 1.0f, 0.5f);
    cudaEventRecord(e0); k_ffma<<<blocks, th>>>(out, it, 1.0f, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    macs = (double)blocks * th * it * 32;
    printf("ffma warps/CTA=%d: %.1f TFLOP/s  (%.0f FMA/clk/SM)\n", warps, 2 * macs / ms / 1e9,
           macs / (ms * 1e-3) / 148 / 1.965e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
