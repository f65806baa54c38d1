// k_marginals.cu -- a1: fixed-point measure of importance (Eq. 1; R1, R7).
//
// q(x) = RNE(phi(x) * 2^S) as int64; x1[i] += q, x2[j] += q, x3[k] += q.  Integer sums are
// exact, so the result does not depend on the launch configuration or atomic order.
//
// Dense layout: X(i,j,k) at base[(k*J + j)*pitch + i].  A "row" is (j,k): `pitch` floats.
// Each thread owns a fixed set of column quads (float4) of every row it visits and keeps
// their x1 partial sums in registers for the whole kernel; row totals (x2[j], x3[k]) are
// reduced across the row's threads (warp shuffles, plus shared memory when a row spans
// several warps).  Grid = a few blocks per SM, each streaming a contiguous row range, so
// the pass is one coalesced sweep over HBM (4 B / entry algorithmic).
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace sbt {

template <int MOI>
__device__ __forceinline__ long long quant(float x, float scf, double scd) {
  if (MOI == 0) {
    return __float2ll_rn(fabsf(x) * scf);      // exact product (power-of-two scale)
  } else {
    const double d = (double)x;
    return __double2ll_rn(__dmul_rn(__dmul_rn(d, d), scd));   // d*d exact (48 bits)
  }
}

template <int VEC> struct VecT;
template <> struct VecT<4> { using T = float4; };
template <> struct VecT<1> { using T = float; };

template <int VEC>
__device__ __forceinline__ typename VecT<VEC>::T ld_stream(const float* p);
template <> __device__ __forceinline__ float4 ld_stream<4>(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
template <> __device__ __forceinline__ float ld_stream<1>(const float* p) { return __ldcs(p); }

__device__ __forceinline__ float comp(const float4& v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}
__device__ __forceinline__ float comp(const float& v, int) { return v; }

constexpr int kMargThreads = 256;
constexpr int kMargWarps = kMargThreads / 32;
constexpr int kX3Slots = 64;

// wpr = warps per row (1, 2, 4, 8); G = 8 / wpr rows in flight per block step.
template <int MOI, int VEC, int V, int UR>
__global__ void __launch_bounds__(kMargThreads) marg_dense_kernel(
    const float* __restrict__ X, int64_t pitch, int I, int J, int64_t row0, int64_t nrows,
    int wpr, int64_t rows_per_block, float scf, double scd, unsigned long long* __restrict__ x1,
    unsigned long long* __restrict__ x2, unsigned long long* __restrict__ x3) {
  __shared__ long long red[2][kMargWarps][UR];
  __shared__ unsigned long long x3s[kX3Slots];
  extern __shared__ unsigned long long x1s[];   // [I] when G > 1
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = kMargWarps / wpr;
  const int g = warp / wpr, wr = warp - g * wpr;
  const int t = wr * 32 + lane;
  const int TPR = wpr * 32;
  const int Q = (int)(pitch / VEC);
  const int64_t rb = (int64_t)blockIdx.x * rows_per_block;
  const int64_t re = min(rb + rows_per_block, nrows);
  if (rb >= re) return;
  const int64_t kfirst = (row0 + rb) / J;
  const bool x3_local = ((row0 + re - 1) / J - kfirst) < kX3Slots;
  for (int s = threadIdx.x; s < kX3Slots; s += blockDim.x) x3s[s] = 0;
  if (G > 1)
    for (int s = threadIdx.x; s < I; s += blockDim.x) x1s[s] = 0;
  __syncthreads();

  long long acc[V][VEC];
#pragma unroll
  for (int c = 0; c < V; ++c)
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[c][e] = 0;

  int buf = 0;
  for (int64_t r0 = rb; r0 < re; r0 += (int64_t)G * UR) {
    typename VecT<VEC>::T v[UR][V];
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const int64_t row = r0 + (int64_t)u * G + g;
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const int qd = t + c * TPR;
        if (row < re && qd < Q) {
          v[u][c] = ld_stream<VEC>(X + (row0 + row) * pitch + (int64_t)qd * VEC);
        } else {
          if constexpr (VEC == 4) v[u][c] = make_float4(0.f, 0.f, 0.f, 0.f);
          else v[u][c] = 0.f;
        }
      }
    }
    long long rs[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      rs[u] = 0;
#pragma unroll
      for (int c = 0; c < V; ++c)
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const long long q = quant<MOI>(comp(v[u][c], e), scf, scd);
          acc[c][e] += q;
          rs[u] += q;
        }
      rs[u] = warp_sum_ll(rs[u]);
    }
    if (wpr == 1) {
      if (lane == 0) {
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const int64_t row = r0 + (int64_t)u * G + g;
          if (row < re && rs[u] != 0) {
            const int64_t gr = row0 + row;
            const int64_t k = gr / J, j = gr - k * J;
            atomicAdd(&x2[j], (unsigned long long)rs[u]);
            if (x3_local) atomicAdd(&x3s[k - kfirst], (unsigned long long)rs[u]);
            else atomicAdd(&x3[k], (unsigned long long)rs[u]);
          }
        }
      }
    } else {
      if (lane == 0) {
#pragma unroll
        for (int u = 0; u < UR; ++u) red[buf][warp][u] = rs[u];
      }
      __syncthreads();
      if (wr == 0 && lane < UR) {
        const int64_t row = r0 + (int64_t)lane * G + g;
        if (row < re) {
          long long s = 0;
          for (int w = 0; w < wpr; ++w) s += red[buf][g * wpr + w][lane];
          if (s != 0) {
            const int64_t gr = row0 + row;
            const int64_t k = gr / J, j = gr - k * J;
            atomicAdd(&x2[j], (unsigned long long)s);
            if (x3_local) atomicAdd(&x3s[k - kfirst], (unsigned long long)s);
            else atomicAdd(&x3[k], (unsigned long long)s);
          }
        }
      }
      buf ^= 1;
    }
  }
  // x1: combine the G row groups in shared memory, then one global atomic per column.
#pragma unroll
  for (int c = 0; c < V; ++c)
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const int col = (t + c * TPR) * VEC + e;
      if (col < I && acc[c][e] != 0) {
        if (G > 1) atomicAdd(&x1s[col], (unsigned long long)acc[c][e]);
        else atomicAdd(&x1[col], (unsigned long long)acc[c][e]);
      }
    }
  __syncthreads();
  if (G > 1)
    for (int s = threadIdx.x; s < I; s += blockDim.x)
      if (x1s[s]) atomicAdd(&x1[s], x1s[s]);
  if (x3_local)
    for (int s = threadIdx.x; s < kX3Slots; s += blockDim.x)
      if (x3s[s]) atomicAdd(&x3[kfirst + s], x3s[s]);
}

static inline float pow2f(int S) { return ldexpf(1.0f, S); }  // exact for S in [-126, 127]

template <int MOI, int VEC, int V>
static cudaError_t marg_launch(const DenseView& X, int64_t row0, int64_t nrows, int wpr,
                               float scf, double scd, unsigned long long* x1,
                               unsigned long long* x2, unsigned long long* x3, cudaStream_t st) {
  constexpr int UR = 2;
  const int G = kMargWarps / wpr;
  const int64_t step = (int64_t)G * UR;
  int64_t nblocks = (int64_t)kNumSMs * 6;
  int64_t rpb = ceil_div(ceil_div(nrows, nblocks), step) * step;
  if (rpb < step) rpb = step;
  nblocks = ceil_div(nrows, rpb);
  const size_t smem = G > 1 ? sizeof(unsigned long long) * (size_t)X.I : 0;
  marg_dense_kernel<MOI, VEC, V, UR><<<(unsigned)nblocks, kMargThreads, smem, st>>>(
      X.base, X.pitch, (int)X.I, (int)X.J, row0, nrows, wpr, rpb, scf, scd, x1, x2, x3);
  return cudaGetLastError();
}

template <int MOI, int VEC>
static cudaError_t marg_dispatch_v(const DenseView& X, int64_t row0, int64_t nrows, float scf,
                                   double scd, unsigned long long* x1, unsigned long long* x2,
                                   unsigned long long* x3, cudaStream_t st) {
  const int64_t Q = X.pitch / VEC;
  // smallest warps-per-row such that V = ceil(Q / (32*wpr)) <= 4
  int wpr = 1;
  while (wpr < 8 && ceil_div(Q, 32 * wpr) > 4) wpr *= 2;
  const int64_t V = ceil_div(Q, 32 * wpr);
  if (V > 4) return cudaErrorInvalidValue;   // rows longer than 4096 (VEC=4) unsupported
  switch (V) {
    case 1: return marg_launch<MOI, VEC, 1>(X, row0, nrows, wpr, scf, scd, x1, x2, x3, st);
    case 2: return marg_launch<MOI, VEC, 2>(X, row0, nrows, wpr, scf, scd, x1, x2, x3, st);
    case 3: return marg_launch<MOI, VEC, 3>(X, row0, nrows, wpr, scf, scd, x1, x2, x3, st);
    default: return marg_launch<MOI, VEC, 4>(X, row0, nrows, wpr, scf, scd, x1, x2, x3, st);
  }
}

cudaError_t launch_marginals_dense(const DenseView& X, int64_t k0, int64_t nk, int moi, int S,
                                   int64_t* x1, int64_t* x2, int64_t* x3, cudaStream_t st) {
  if (nk <= 0 || X.I <= 0 || X.J <= 0) return cudaSuccess;
  const int64_t row0 = k0 * X.J, nrows = nk * X.J;
  const float scf = pow2f(S < -126 ? -126 : (S > 127 ? 127 : S));
  const double scd = ldexp(1.0, S);
  auto* u1 = reinterpret_cast<unsigned long long*>(x1);
  auto* u2 = reinterpret_cast<unsigned long long*>(x2);
  auto* u3 = reinterpret_cast<unsigned long long*>(x3);
  const bool vec4 = (X.pitch % 4 == 0) && ((uintptr_t)X.base % 16 == 0);
  if (moi == 0) {
    return vec4 ? marg_dispatch_v<0, 4>(X, row0, nrows, scf, scd, u1, u2, u3, st)
                : marg_dispatch_v<0, 1>(X, row0, nrows, scf, scd, u1, u2, u3, st);
  }
  return vec4 ? marg_dispatch_v<1, 4>(X, row0, nrows, scf, scd, u1, u2, u3, st)
              : marg_dispatch_v<1, 1>(X, row0, nrows, scf, scd, u1, u2, u3, st);
}

// ---------------------------------------------------------------------------------------
// COO marginals: one thread per stored entry.  Entries are sorted by (k, j, i), so x3 is
// aggregated over runs of equal k inside a warp before its atomic.
// ---------------------------------------------------------------------------------------
template <int MOI>
__global__ void marg_coo_kernel(const int32_t* __restrict__ ii, const int32_t* __restrict__ jj,
                                const int32_t* __restrict__ kk, const float* __restrict__ vv,
                                int64_t nnz, float scf, double scd, unsigned long long* x1,
                                unsigned long long* x2, unsigned long long* x3) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < nnz;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = base + threadIdx.x;
    long long q = 0;
    int k = -1;
    if (n < nnz) {
      q = quant<MOI>(vv[n], scf, scd);
      if (q) {
        atomicAdd(&x1[ii[n]], (unsigned long long)q);
        atomicAdd(&x2[jj[n]], (unsigned long long)q);
      }
      k = kk[n];
    }
    // segmented reduction of q over equal k within the warp
    const unsigned same = __match_any_sync(0xffffffffu, k);
    const int leader = __ffs(same) - 1;
    long long s = 0;
    for (unsigned m = same; m; m &= m - 1) {
      const int src = __ffs(m) - 1;
      s += __shfl_sync(same, q, src);
    }
    if (lane == leader && k >= 0 && s) atomicAdd(&x3[k], (unsigned long long)s);
  }
}

// Replicated variant for large stores (C5: Zipf-hot indices).  The hottest index of a Zipf(1.2)
// mode takes ~2 % of all entries; their int64 reds on one address serialise in its L2 slice
// (~2 M of them at C5, ~2.5 ms).  Block b adds into replica b mod nrep of x1 and x2 (nrep
// addresses per index in different slices), runs of equal j and k are combined first (entries
// are sorted by (k, j, i)), and a second kernel adds the replicas into x1 / x2 (integer sums:
// exact in any order).
template <int MOI, bool VEC>
__global__ void __launch_bounds__(256) marg_coo_rep_kernel(
    const int32_t* __restrict__ ii, const int32_t* __restrict__ jj, const int32_t* __restrict__ kk,
    const float* __restrict__ vv, int64_t nnz, float scf, double scd, unsigned long long* __restrict__ x1r,
    unsigned long long* __restrict__ x2r, int64_t I, int64_t J, int nrep, unsigned long long* __restrict__ x3) {
  const int lane = threadIdx.x & 31;
  const int rp = blockIdx.x % nrep;
  unsigned long long* x1 = x1r + (int64_t)rp * I;
  unsigned long long* x2 = x2r + (int64_t)rp * J;
  const int64_t step = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x) * 4; base < nnz; base += step) {
    const int64_t e0 = base + 4 * (int64_t)threadIdx.x;
    int i[4], j[4], k[4];
    long long q[4];
    if (VEC && e0 + 3 < nnz) {
      const int4 a = __ldcs(reinterpret_cast<const int4*>(ii + e0));
      const int4 b = __ldcs(reinterpret_cast<const int4*>(jj + e0));
      const int4 c = __ldcs(reinterpret_cast<const int4*>(kk + e0));
      const float4 v = __ldcs(reinterpret_cast<const float4*>(vv + e0));
      i[0] = a.x; i[1] = a.y; i[2] = a.z; i[3] = a.w;
      j[0] = b.x; j[1] = b.y; j[2] = b.z; j[3] = b.w;
      k[0] = c.x; k[1] = c.y; k[2] = c.z; k[3] = c.w;
      q[0] = quant<MOI>(v.x, scf, scd); q[1] = quant<MOI>(v.y, scf, scd);
      q[2] = quant<MOI>(v.z, scf, scd); q[3] = quant<MOI>(v.w, scf, scd);
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int64_t e = e0 + t;
        const bool in = e < nnz;
        i[t] = in ? __ldcs(ii + e) : 0;
        j[t] = in ? __ldcs(jj + e) : (t ? j[t - 1] : 0);
        k[t] = in ? __ldcs(kk + e) : (t ? k[t - 1] : -1);
        q[t] = in ? quant<MOI>(__ldcs(vv + e), scf, scd) : 0;
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (q[t]) atomicAdd(&x1[i[t]], (unsigned long long)q[t]);
    // x2: runs of equal j among the thread's 4 entries
    long long s = q[0];
#pragma unroll
    for (int t = 1; t < 4; ++t) {
      if (j[t] != j[t - 1]) {
        if (s) atomicAdd(&x2[j[t - 1]], (unsigned long long)s);
        s = 0;
      }
      s += q[t];
    }
    if (s) atomicAdd(&x2[j[3]], (unsigned long long)s);
    // x3: one slice for the thread and the warp -> one REDUX sum; else per-thread runs
    const int k0 = __shfl_sync(0xffffffffu, k[0], 0);
    const bool one = k[0] == k[3] && k[0] == k0 && k0 >= 0;
    const long long st = q[0] + q[1] + q[2] + q[3];
    if (__all_sync(0xffffffffu, one)) {
      const unsigned long long u = (unsigned long long)st;   // < 2^63: 21 + 21 + 21 bit chunks
      const unsigned c0 = __reduce_add_sync(0xffffffffu, (unsigned)(u & 0x1fffffu));
      const unsigned c1 = __reduce_add_sync(0xffffffffu, (unsigned)((u >> 21) & 0x1fffffu));
      const unsigned c2 = __reduce_add_sync(0xffffffffu, (unsigned)(u >> 42));
      const unsigned long long tot = (unsigned long long)c0 + ((unsigned long long)c1 << 21) + ((unsigned long long)c2 << 42);
      if (lane == 0 && tot) atomicAdd(&x3[k0], tot);
    } else {
      long long r3 = q[0];
#pragma unroll
      for (int t = 1; t < 4; ++t) {
        if (k[t] != k[t - 1]) {
          if (r3 && k[t - 1] >= 0) atomicAdd(&x3[k[t - 1]], (unsigned long long)r3);
          r3 = 0;
        }
        r3 += q[t];
      }
      if (r3 && k[3] >= 0) atomicAdd(&x3[k[3]], (unsigned long long)r3);
    }
  }
}

__global__ void marg_rep_combine_kernel(const unsigned long long* __restrict__ rep, int64_t n, int nrep,
                                        unsigned long long* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long s = 0;
    for (int t = 0; t < nrep; ++t) s += rep[(int64_t)t * n + e];
    if (s) out[e] += s;
  }
}

int marg_coo_replicas(int64_t nnz, int64_t I, int64_t J) {
  if (getenv("SAMBATEN_COO_MARG_NOREP")) return 1;
  if (const char* e = getenv("SBT_MARG_NREP")) return atoi(e);
  const int64_t cap = nnz / (4 * std::max<int64_t>(I + J, 1));   // zeroing + combining <= 1/4 of the pass's entries
  return (int)std::min<int64_t>(kMargCooMaxRep, cap);
}

cudaError_t launch_marginals_coo(const int32_t* i, const int32_t* j, const int32_t* k,
                                 const float* v, int64_t nnz, int moi, int S, int64_t* x1,
                                 int64_t* x2, int64_t* x3, cudaStream_t st, int64_t I, int64_t J,
                                 int64_t* rep_ws, int nrep) {
  if (nnz <= 0) return cudaSuccess;
  const float scf = pow2f(S < -126 ? -126 : (S > 127 ? 127 : S));
  const double scd = ldexp(1.0, S);
  if (rep_ws && nrep >= 2 && I > 0 && J > 0) {
    auto* r1 = reinterpret_cast<unsigned long long*>(rep_ws);
    auto* r2 = r1 + (int64_t)nrep * I;
    cudaError_t e = cudaMemsetAsync(rep_ws, 0, sizeof(int64_t) * (size_t)nrep * (I + J), st);
    if (e != cudaSuccess) return e;
    const char* bps = getenv("SBT_MARG_BPS");
    const int blocks = kNumSMs * (bps ? atoi(bps) : 16);   // 16 per SM measured best (C5 probe)
    auto* u3 = reinterpret_cast<unsigned long long*>(x3);
    const bool vec = ((uintptr_t)i | (uintptr_t)j | (uintptr_t)k | (uintptr_t)v) % 16 == 0;
    if (moi == 0 && vec)
      marg_coo_rep_kernel<0, true><<<blocks, 256, 0, st>>>(i, j, k, v, nnz, scf, scd, r1, r2, I, J, nrep, u3);
    else if (moi == 0)
      marg_coo_rep_kernel<0, false><<<blocks, 256, 0, st>>>(i, j, k, v, nnz, scf, scd, r1, r2, I, J, nrep, u3);
    else if (vec)
      marg_coo_rep_kernel<1, true><<<blocks, 256, 0, st>>>(i, j, k, v, nnz, scf, scd, r1, r2, I, J, nrep, u3);
    else
      marg_coo_rep_kernel<1, false><<<blocks, 256, 0, st>>>(i, j, k, v, nnz, scf, scd, r1, r2, I, J, nrep, u3);
    marg_rep_combine_kernel<<<(unsigned)std::min<int64_t>(ceil_div(I, 256), kNumSMs * 4), 256, 0, st>>>(r1, I, nrep, reinterpret_cast<unsigned long long*>(x1));
    marg_rep_combine_kernel<<<(unsigned)std::min<int64_t>(ceil_div(J, 256), kNumSMs * 4), 256, 0, st>>>(r2, J, nrep, reinterpret_cast<unsigned long long*>(x2));
    return cudaGetLastError();
  }
  const int threads = 256;
  int64_t blocks = ceil_div(nnz, threads);
  if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
  auto* u1 = reinterpret_cast<unsigned long long*>(x1);
  auto* u2 = reinterpret_cast<unsigned long long*>(x2);
  auto* u3 = reinterpret_cast<unsigned long long*>(x3);
  if (moi == 0)
    marg_coo_kernel<0><<<(unsigned)blocks, threads, 0, st>>>(i, j, k, v, nnz, scf, scd, u1, u2, u3);
  else
    marg_coo_kernel<1><<<(unsigned)blocks, threads, 0, st>>>(i, j, k, v, nnz, scf, scd, u1, u2, u3);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// max phi (fixed-point range, R7)
// ---------------------------------------------------------------------------------------
template <int MOI>
__device__ __forceinline__ double phi_d(float x) {
  const double d = (double)x;
  return MOI == 0 ? fabs(d) : d * d;
}

// max phi(x) = phi(max |x|) (phi monotone in |x|): the scan keeps max |x| in fp32 (exact) and
// converts once.  Rows (pitch-strided) are walked by a warp each, float4 when aligned.
template <int MOI>
__device__ __forceinline__ void flush_max(float mx, unsigned long long* out) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const double m = phi_d<MOI>(mx);
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

template <int MOI>
__global__ void max_phi_dense_kernel(const float* __restrict__ X, int64_t pitch, int64_t I,
                                     int64_t row0, int64_t nrows, unsigned long long* out) {
  float mx = 0.f;
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (pitch % 4) == 0 && (((uintptr_t)X) & 15) == 0;
  for (int64_t row = wid; row < nrows; row += nw) {
    const float* p = X + (row0 + row) * pitch;
    if (vec) {
      const int64_t n4 = I / 4;
      for (int64_t c = lane; c < n4; c += 32) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(p) + c);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
      for (int64_t c = 4 * n4 + lane; c < I; c += 32) mx = fmaxf(mx, fabsf(p[c]));
    } else {
      for (int64_t c = lane; c < I; c += 32) mx = fmaxf(mx, fabsf(p[c]));
    }
  }
  flush_max<MOI>(mx, out);
}

// a0 fused: copy a contiguous device batch into the store (contiguous: pitch == I) and
// track max |x| in the same pass (16 B vectors; n4 = floats / 4).
template <int MOI>
__global__ void ingest_dense_kernel(const float4* __restrict__ src, float4* __restrict__ dst, int64_t n4,
                                    unsigned long long* out) {
  float mx = 0.f;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(src + e);
    __stcg(dst + e, v);
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  flush_max<MOI>(mx, out);
}

template <int MOI>
__global__ void max_phi_vals_kernel(const float* __restrict__ v, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, phi_d<MOI>(v[e]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0)
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

cudaError_t launch_ingest_dense(const float* src, float* dst, int64_t n, int moi, unsigned long long* out,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = ceil_div(n / 4, 256);
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  if (blocks < 1) blocks = 1;
  auto* s4 = reinterpret_cast<const float4*>(src);
  auto* d4 = reinterpret_cast<float4*>(dst);
  if (moi == 0) ingest_dense_kernel<0><<<(unsigned)blocks, 256, 0, st>>>(s4, d4, n / 4, out);
  else ingest_dense_kernel<1><<<(unsigned)blocks, 256, 0, st>>>(s4, d4, n / 4, out);
  return cudaGetLastError();
}

cudaError_t launch_max_phi_dense(const DenseView& X, int64_t k0, int64_t nk, int moi,
                                 unsigned long long* out, cudaStream_t st) {
  const int64_t nrows = nk * X.J;
  if (nrows <= 0) return cudaSuccess;
  int64_t blocks = ceil_div(nrows, 8);   // a warp per row, 8 warps per block
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  if (moi == 0)
    max_phi_dense_kernel<0><<<(unsigned)blocks, 256, 0, st>>>(X.base, X.pitch, X.I, k0 * X.J, nrows, out);
  else
    max_phi_dense_kernel<1><<<(unsigned)blocks, 256, 0, st>>>(X.base, X.pitch, X.I, k0 * X.J, nrows, out);
  return cudaGetLastError();
}

cudaError_t launch_max_phi_vals(const float* v, int64_t n, int moi, unsigned long long* out,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = ceil_div(n, 256);
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  if (moi == 0) max_phi_vals_kernel<0><<<(unsigned)blocks, 256, 0, st>>>(v, n, out);
  else max_phi_vals_kernel<1><<<(unsigned)blocks, 256, 0, st>>>(v, n, out);
  return cudaGetLastError();
}

}  // namespace sbt
