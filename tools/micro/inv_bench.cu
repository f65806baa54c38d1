// Microbenchmark (dev tool): cycles of one warp's 10 x 10 SPD inverse variants.
#include <cstdio>
#include <cuda_runtime.h>
// Register Gauss-Jordan for R <= RB <= 16: lane c < 2R holds column c of [V | I] in
// registers; step j broadcasts the pivot and the R entries of column j by shuffles.
template <int RB>
__device__ __forceinline__ bool sbt_inv(const double* V, double* Vi, int R) {
  const int lane = threadIdx.x & 31;
  double col[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    double v = 0.0;
    if (i < R) v = lane < R ? V[i * R + lane] : (lane - R == i ? 1.0 : 0.0);
    col[i] = v;
  }
  bool ok = true;
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    if (j < R) {
      const double piv = __shfl_sync(0xffffffffu, col[j], j);
      ok = ok && (piv > 0.0);
      double fcol[RB];
#pragma unroll
      for (int i = 0; i < RB; ++i) fcol[i] = __shfl_sync(0xffffffffu, col[i], j);
      col[j] = col[j] / piv;
#pragma unroll
      for (int i = 0; i < RB; ++i)
        if (i < R && i != j) col[i] = fma(-fcol[i], col[j], col[i]);
    }
  }
  if (ok && lane >= R && lane < 2 * R)
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if (i < R) Vi[i * R + (lane - R)] = col[i];
  __syncwarp();
  return ok;
}


// variant: reciprocal once per step (MUFU + Newton), no IEEE division
template <int RB>
__device__ __forceinline__ bool inv_rcp(const double* V, double* Vi, int R) {
  const int lane = threadIdx.x & 31;
  double col[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    double v = 0.0;
    if (i < R) v = lane < R ? V[i * R + lane] : (lane - R == i ? 1.0 : 0.0);
    col[i] = v;
  }
  bool ok = true;
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    if (j < R) {
      double fcol[RB];
#pragma unroll
      for (int i = 0; i < RB; ++i) fcol[i] = __shfl_sync(0xffffffffu, col[i], j);
      const double piv = fcol[j];
      ok = ok && (piv > 0.0);
      double r = __drcp_rn(piv);
      col[j] = col[j] * r;
#pragma unroll
      for (int i = 0; i < RB; ++i)
        if (i < R && i != j) col[i] = fma(-fcol[i], col[j], col[i]);
    }
  }
  if (ok && lane >= R && lane < 2 * R)
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if (i < R) Vi[i * R + (lane - R)] = col[i];
  __syncwarp();
  return ok;
}

template <int V>
__global__ void k(const double* Vg, double* out, long long* cyc, int reps) {
  __shared__ double Vs[100], Vi[100];
  for (int e = threadIdx.x; e < 100; e += 32) Vs[e] = Vg[e];
  __syncwarp();
  long long t0 = clock64();
  bool ok = true;
  for (int r = 0; r < reps; ++r) {
    if (V == 0) ok &= sbt_inv<10>(Vs, Vi, 10);
    else ok &= inv_rcp<10>(Vs, Vi, 10);
    Vs[threadIdx.x % 10] += 1e-30 * Vi[threadIdx.x % 10];
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[V] = (t1 - t0) / reps; out[0] = Vi[0] + ok; }
}

int main() {
  double h[100];
  for (int i = 0; i < 10; ++i) for (int j = 0; j < 10; ++j) h[i * 10 + j] = (i == j ? 2.0 : 0.0) + 0.3 / (1 + i + j);
  double *d, *o; long long* c; cudaMalloc(&d, 800); cudaMalloc(&o, 8); cudaMalloc(&c, 16);
  cudaMemcpy(d, h, 800, cudaMemcpyHostToDevice);
  k<0><<<1, 32>>>(d, o, c, 100); k<1><<<1, 32>>>(d, o, c, 100); cudaDeviceSynchronize();
  long long hc[2]; cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
  printf("register GJ (division): %lld cycles; reciprocal: %lld cycles; err=%s\n", hc[0], hc[1], cudaGetErrorString(cudaGetLastError()));
}
