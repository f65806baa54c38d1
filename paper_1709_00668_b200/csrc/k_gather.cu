// k_gather.cu -- a3 (dense): the summaries X_s = X(I_s, J_s, K_s U new).
//
// Y[rep][u][q][p] = X(Is[p], Js[q], Kp[u]) and, for the cluster ALS, its per-slice transpose
// Yt[rep][u][p][q].  Block = (32-row q tile, (rep, slice u) pair); for each 32-column p tile the
// 8 warps gather 4 source rows each (lanes walk the sorted I_s list held in shared memory,
// so neighbouring lanes share 32 B sectors of the source row), write the Y rows coalesced
// and stage the 32 x 32 block in shared memory (padded, conflict-free) for the coalesced Yt
// rows.  Pure data movement: both layouts are bit-exact copies.
#include "common.cuh"
#include "internal.h"

namespace sbt {

constexpr int kGatherThreads = 256;

// The (rep, u) pairs of all summaries ordered by their source slice K'[rep][u] (ties by rep:
// stable), so the gather's blocks walk the store slice by slice -- the 16 repetitions' reads of
// a new slice hit L2 after the first and the address translations stay within a few slices of
// the 108 GB store (random slice order missed the TLB).  One block: a bitmask per slice of the
// repetitions that sampled it (a repetition's K' holds distinct slices), an exclusive scan of
// the popcounts, and pair (rep, u) goes to start[k] + popc(mask[k] & ((1 << rep) - 1)).  Exact
// integer work, independent of thread order.
constexpr int kOrderSlices = 8192;   // slices of the store covered (2 x 32 KB of dynamic shared memory)
__global__ void __launch_bounds__(1024) gather_order_kernel(const int32_t* __restrict__ Kp, int nK, int r,
                                                            int64_t sK, int nslices, int32_t* __restrict__ order) {
  extern __shared__ unsigned order_sm[];   // [nslices] masks | [nslices] starts
  unsigned* mask = order_sm;
  int* start = reinterpret_cast<int*>(order_sm + nslices);
  __shared__ int sh[33];
  __shared__ int carry;
  for (int k = threadIdx.x; k < nslices; k += blockDim.x) mask[k] = 0u;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < nK * r; e += blockDim.x) {
    const int rep = e / nK, u = e - rep * nK;
    atomicOr(&mask[Kp[rep * sK + u]], 1u << rep);
  }
  __syncthreads();
  for (int k0 = 0; k0 < nslices; k0 += blockDim.x) {   // exclusive scan of the popcounts
    const int k = k0 + threadIdx.x;
    int tot;
    const int ex = block_excl_scan(k < nslices ? __popc(mask[k]) : 0, sh, &tot);
    if (k < nslices) start[k] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nK * r; e += blockDim.x) {
    const int rep = e / nK, u = e - rep * nK;
    const int k = Kp[rep * sK + u];
    order[start[k] + __popc(mask[k] & ((1u << rep) - 1u))] = e;
  }
}

__global__ void __launch_bounds__(kGatherThreads) gather_dense_kernel(
    const float* __restrict__ X, int64_t J, int64_t pitch, const int32_t* __restrict__ Is,
    const int32_t* __restrict__ Js, const int32_t* __restrict__ Kp, int nI, int nJ, int nK,
    int64_t sI, int64_t sJ, int64_t sK, float* __restrict__ Y, float* __restrict__ Yt,
    int64_t y_stride, int pI, int pJ, const int32_t* __restrict__ order) {
  extern __shared__ int32_t is_sh[];
  __shared__ float tile[2][32][33];
  // grid (q tile, pair): pairs in source-slice order when `order` is given, else (rep, slice)
  const int qt = blockIdx.x;
  const int pr = order ? order[blockIdx.y] : (int)blockIdx.y;
  const int rep = pr / nK, u = pr - rep * nK;
  const int32_t* is = Is + rep * sI;
  for (int p = threadIdx.x; p < nI; p += blockDim.x) is_sh[p] = is[p];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = qt * 32;
  const int nq = min(32, nJ - q0);
  const int32_t* js = Js + rep * sJ;
  const int64_t ku = Kp[rep * sK + u];
  float* Ys = Y + rep * y_stride + (int64_t)u * nJ * pI;
  float* Yts = Yt ? Yt + rep * y_stride + (int64_t)u * nI * pJ : nullptr;
  const float* srow[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int ql = warp * 4 + k;
    srow[k] = ql < nq ? X + (ku * J + js[q0 + ql]) * pitch : nullptr;
  }
  // two 32-column tiles per step: 8 independent gathers in flight per thread, one barrier pair
  for (int p0 = 0; p0 < pI; p0 += 64) {
    float v[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int p = p0 + 32 * h + lane;
#pragma unroll
      for (int k = 0; k < 4; ++k) v[h][k] = (srow[k] && p < nI) ? __ldg(srow[k] + is_sh[p]) : 0.f;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int p = p0 + 32 * h + lane;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int ql = warp * 4 + k;
        if (srow[k] && p < pI) Ys[(int64_t)(q0 + ql) * pI + p] = v[h][k];   // zero pad p >= nI
        tile[h][ql][lane] = v[h][k];
      }
    }
    if (Yts) {
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int pl = warp * 4 + k;   // p offset within the tile
          const int pp = p0 + 32 * h + pl;
          if (pp < nI && q0 + lane < pJ)
            Yts[(int64_t)pp * pJ + q0 + lane] = lane < nq ? tile[h][lane][pl] : 0.f;
        }
      __syncthreads();
    }
  }
}

cudaError_t launch_gather_dense(const DenseView& X, const int32_t* Is, const int32_t* Js,
                                const int32_t* Kp, int nI, int nJ, int nK, int r,
                                int64_t sI, int64_t sJ, int64_t sK, float* Y, int64_t y_stride,
                                cudaStream_t st, float* Yt, int pI, int pJ, int32_t* order_ws, int64_t nslices) {
  if (nK <= 0 || nJ <= 0 || nI <= 0 || r <= 0) return cudaSuccess;
  if (pI < nI) pI = nI;
  if (pJ < nJ) pJ = nJ;
  const int npair = nK * r;
  if (npair > 65535) return cudaErrorInvalidConfiguration;   // grid.y limit
  const int32_t* order = nullptr;
  if (order_ws && nslices > 0 && nslices <= kOrderSlices && r > 1 && r <= 32) {
    const int smem = (int)(2 * sizeof(int) * nslices);
    cudaFuncSetAttribute(gather_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4 * kOrderSlices);
    gather_order_kernel<<<1, 1024, smem, st>>>(Kp, nK, r, sK, (int)nslices, order_ws);
    order = order_ws;
  }
  dim3 grid((unsigned)ceil_div(pJ, 32), (unsigned)npair, 1);
  gather_dense_kernel<<<grid, kGatherThreads, sizeof(int32_t) * nI, st>>>(
      X.base, X.J, X.pitch, Is, Js, Kp, nI, nJ, nK, sI, sJ, sK, Y, Yt, y_stride, pI, pJ, order);
  return cudaGetLastError();
}

}  // namespace sbt
