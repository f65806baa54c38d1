// k_gather.cu -- a3 (dense): the summaries X_s = X(I_s, J_s, K_s U new).
//
// Y[rep][u][q][p] = X(Is[p], Js[q], Kp[u]).  One warp per output row (rep, u, q): the lanes
// walk the sorted I_s list (held in shared memory for the block's repetition) and load
// X at those columns of source row (Kp[u], Js[q]).  Sorted indices make neighbouring lanes
// share 32 B sectors; output rows are written contiguously.  Pure data movement: the
// summary is a bit-exact copy.
#include "common.cuh"
#include "internal.h"

namespace sbt {

constexpr int kGatherThreads = 256;

__global__ void __launch_bounds__(kGatherThreads) gather_dense_kernel(
    const float* __restrict__ X, int64_t J, int64_t pitch, const int32_t* __restrict__ Is,
    const int32_t* __restrict__ Js, const int32_t* __restrict__ Kp, int nI, int nJ, int nK,
    int64_t sI, int64_t sJ, int64_t sK, float* __restrict__ Y, int64_t y_stride,
    int rows_per_block) {
  extern __shared__ int32_t is_sh[];
  const int rep = blockIdx.y;
  const int32_t* is = Is + rep * sI;
  for (int p = threadIdx.x; p < nI; p += blockDim.x) is_sh[p] = is[p];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nrows = (int64_t)nK * nJ;
  const int64_t rb = (int64_t)blockIdx.x * rows_per_block;
  const int64_t re = min(rb + rows_per_block, nrows);
  float* Yr = Y + rep * y_stride;
  const int32_t* js = Js + rep * sJ;
  const int32_t* kp = Kp + rep * sK;
  for (int64_t row = rb + warp; row < re; row += kGatherThreads / 32) {
    const int u = (int)(row / nJ), q = (int)(row - (int64_t)u * nJ);
    const float* src = X + ((int64_t)kp[u] * J + js[q]) * pitch;
    float* dst = Yr + row * nI;
    for (int p = lane; p < nI; p += 32) dst[p] = __ldg(src + is_sh[p]);
  }
}

cudaError_t launch_gather_dense(const DenseView& X, const int32_t* Is, const int32_t* Js,
                                const int32_t* Kp, int nI, int nJ, int nK, int r,
                                int64_t sI, int64_t sJ, int64_t sK, float* Y, int64_t y_stride,
                                cudaStream_t st) {
  const int64_t nrows = (int64_t)nK * nJ;
  if (nrows <= 0 || nI <= 0 || r <= 0) return cudaSuccess;
  // ~4 waves of 256-thread blocks over the chip, at least 8 rows (one per warp) per block
  int64_t want = (int64_t)kNumSMs * 8 / r;
  if (want < 1) want = 1;
  int64_t rpb = ceil_div(nrows, want);
  if (rpb < 8) rpb = 8;
  const int64_t nb = ceil_div(nrows, rpb);
  dim3 grid((unsigned)nb, (unsigned)r);
  gather_dense_kernel<<<grid, kGatherThreads, sizeof(int32_t) * nI, st>>>(
      X.base, X.J, X.pitch, Is, Js, Kp, nI, nJ, nK, sI, sJ, sK, Y, y_stride, (int)rpb);
  return cudaGetLastError();
}

}  // namespace sbt
