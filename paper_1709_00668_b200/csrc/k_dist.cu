// k_dist.cu -- data movement of the time-slab sharded update (DESIGN.md
// "Multi-GPU").  Every rank holds the frontal slices it ingested; a repetition's summary is
// assembled on its owner (rep rho on rank rho mod G) from the slices of every rank:
//   slice_gather_kernel  one job = one summary slice u of one repetition: the I_s x J_s
//                        sub-slice of a LOCAL store slice, written as a Y slice [q][p] (pitch
//                        pI) and optionally its transpose Yt [p][q] (pitch pJ), either into
//                        the repetition's own buffer (owned here) or packed into a send buffer;
//   slice_copy_kernel    unpack received packed slices into the owner's Y / Yt at their u;
//   x3_scatter_kernel    local mode-3 marginals -> their global slice positions.
#include "common.cuh"
#include "internal.h"

namespace sbt {

namespace {

constexpr int kDT = 256;

__global__ void __launch_bounds__(kDT) slice_gather_kernel(const float* __restrict__ X, int64_t J,
                                                           int64_t pitch, const SliceJob* __restrict__ jobs,
                                                           const int32_t* __restrict__ Is_all,
                                                           const int32_t* __restrict__ Js_all, int nI,
                                                           int nJ, int pI, int pJ) {
  extern __shared__ int32_t is_sh[];
  __shared__ float tile[32][33];
  const SliceJob jb = jobs[blockIdx.y];
  const int qt = blockIdx.x;
  const int32_t* is = Is_all + (int64_t)jb.rep * nI;
  for (int p = threadIdx.x; p < nI; p += blockDim.x) is_sh[p] = is[p];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = qt * 32;
  const int nq = min(32, nJ - q0);
  const int32_t* js = Js_all + (int64_t)jb.rep * nJ;
  const float* srow[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int ql = warp * 4 + k;
    srow[k] = ql < nq ? X + ((int64_t)jb.k_local * J + js[q0 + ql]) * pitch : nullptr;
  }
  for (int p0 = 0; p0 < pI; p0 += 32) {
    const int p = p0 + lane;
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (srow[k] && p < nI) ? __ldg(srow[k] + is_sh[p]) : 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int ql = warp * 4 + k;
      if (srow[k] && p < pI) jb.dY[(int64_t)(q0 + ql) * pI + p] = v[k];
      tile[ql][lane] = v[k];
    }
    if (jb.dYt) {
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int pl = warp * 4 + k;
        if (p0 + pl < nI && q0 + lane < pJ)
          jb.dYt[(int64_t)(p0 + pl) * pJ + q0 + lane] = lane < nq ? tile[lane][pl] : 0.f;
      }
      __syncthreads();
    }
  }
}

__global__ void slice_copy_kernel(const CopyJob* __restrict__ jobs, int64_t nY, int64_t nYt) {
  const CopyJob jb = jobs[blockIdx.y];
  const int64_t n = nY + (jb.dYt ? nYt : 0);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float v = jb.src[e];
    if (e < nY) jb.dY[e] = v;
    else jb.dYt[e - nY] = v;
  }
}

// byte copies of a list of (src, dst, bytes) jobs, 4-byte granularity (bytes % 4 == 0)
__global__ void multi_copy_kernel(const CopyBytes* __restrict__ jobs) {
  const CopyBytes jb = jobs[blockIdx.y];
  const int64_t n = jb.bytes / 4;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(jb.src);
  uint32_t* dst = reinterpret_cast<uint32_t*>(jb.dst);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

__global__ void x3_scatter_kernel(const int64_t* __restrict__ x3l, const int32_t* __restrict__ kmap,
                                  int64_t n, int64_t* __restrict__ x3g) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x)
    x3g[kmap[l]] = x3l[l];
}

__global__ void add_i64_kernel(int64_t* __restrict__ dst, const int64_t* __restrict__ src, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] += src[e];
}

// COO sharded gather: per-rep membership / local-index maps over this rank's LOCAL slices.
// kg = kmap[kl]; mKl[kl] = mK[kg] (bit rho: slice sampled in rep rho, new slices every rep);
// locKl[rho][kl] = u of slice kg in rep rho's K' (locK for old slices, nKs + kg - Ko for new).
__global__ void local_kmaps_kernel(const int32_t* __restrict__ kmap, int64_t Kl, const uint32_t* __restrict__ mK,
                                   const int32_t* __restrict__ locK, int64_t Ko, int nKs, int r,
                                   uint32_t* __restrict__ mKl, int32_t* __restrict__ locKl) {
  for (int64_t kl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; kl < Kl; kl += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kg = kmap[kl];
    mKl[kl] = mK[kg];
    for (int rho = 0; rho < r; ++rho)
      locKl[(int64_t)rho * Kl + kl] = kg < Ko ? locK[(int64_t)rho * Ko + kg] : (int32_t)(nKs + (kg - Ko));
  }
}

}  // namespace

cudaError_t launch_local_kmaps(const int32_t* kmap, int64_t Kl, const uint32_t* mK, const int32_t* locK, int64_t Ko,
                               int nKs, int r, uint32_t* mKl, int32_t* locKl, cudaStream_t st) {
  if (Kl <= 0) return cudaSuccess;
  const int64_t b = ceil_div(Kl, kDT);
  local_kmaps_kernel<<<(unsigned)(b < 1024 ? b : 1024), kDT, 0, st>>>(kmap, Kl, mK, locK, Ko, nKs, r, mKl, locKl);
  return cudaGetLastError();
}

cudaError_t launch_add_i64(int64_t* dst, const int64_t* src, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t b = ceil_div(n, kDT);
  add_i64_kernel<<<(unsigned)(b < 1024 ? b : 1024), kDT, 0, st>>>(dst, src, n);
  return cudaGetLastError();
}

cudaError_t launch_slice_gather(const DenseView& X, const SliceJob* jobs, int njobs, const int32_t* Is_all,
                                const int32_t* Js_all, int nI, int nJ, int pI, int pJ, cudaStream_t st) {
  if (njobs <= 0) return cudaSuccess;
  dim3 grid((unsigned)ceil_div(pJ, 32), (unsigned)njobs);
  slice_gather_kernel<<<grid, kDT, sizeof(int32_t) * nI, st>>>(X.base, X.J, X.pitch, jobs, Is_all, Js_all,
                                                                nI, nJ, pI, pJ);
  return cudaGetLastError();
}

cudaError_t launch_slice_copy(const CopyJob* jobs, int njobs, int64_t nY, int64_t nYt, cudaStream_t st) {
  if (njobs <= 0) return cudaSuccess;
  int64_t bx = ceil_div(nY + nYt, kDT * 4);
  if (bx > 64) bx = 64;
  slice_copy_kernel<<<dim3((unsigned)bx, (unsigned)njobs), kDT, 0, st>>>(jobs, nY, nYt);
  return cudaGetLastError();
}

cudaError_t launch_multi_copy(const CopyBytes* jobs, int njobs, int64_t max_bytes, cudaStream_t st) {
  if (njobs <= 0) return cudaSuccess;
  int64_t bx = ceil_div(max_bytes / 4, kDT * 4);
  if (bx < 1) bx = 1;
  if (bx > 64) bx = 64;
  multi_copy_kernel<<<dim3((unsigned)bx, (unsigned)njobs), kDT, 0, st>>>(jobs);
  return cudaGetLastError();
}

cudaError_t launch_x3_scatter(const int64_t* x3l, const int32_t* kmap, int64_t n, int64_t* x3g,
                              cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  x3_scatter_kernel<<<(unsigned)(ceil_div(n, kDT) < 1024 ? ceil_div(n, kDT) : 1024), kDT, 0, st>>>(x3l, kmap, n, x3g);
  return cudaGetLastError();
}

}  // namespace sbt
