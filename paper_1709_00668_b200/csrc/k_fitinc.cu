// k_fitinc.cu -- a7 without a pass over the whole tensor: the exact fit of the committed model
// kept up to date from one update to the next.
//
// The fit needs <X, M> = sum_f lam_f P[f] with the per-component inner products
//     P[f] = sum_{i,j,k} X(i,j,k) A(i,f) B(j,f) C(k,f),
// plus ||X||^2 and ||M||^2 = lam^T (A^T A * B^T B * C^T C) lam (Grams: cheap).  An update
// appends K_n slices and replaces (A, B, C) by (A', B', C') (C' has K_n more rows).  By the
// telescoping identity A'B'C' - ABC = (A'-A) B' C' + A (B'-B) C' + A B (C'-C) (per component,
// per entry) the new inner products over the OLD slices differ from P only through the rows
// the merge changed:
//     P'[f] = P[f] + sum_{new slices k} sum_{i,j} X A' B' C'
//                  + sum_{j: B'(j,.) != B(j,.)} sum_{old k} sum_i X(i,j,k) A(i,f) (B'-B)(j,f) C'(k,f)
//                  + sum_{k old: C'(k,.) != C(k,.)} sum_j sum_i X(i,j,k) A(i,f) B(j,f) (C'-C)(k,f)
// when A' = A (an A row change would need its whole mode-0 fibre: a full pass instead).  With
// the paper's merge (update zero entries only) old rows change only where the model
// had exact zeros, so after a dense initial model every update takes the first two terms:
// O(batch) bytes instead of the whole tensor.  ||X'||^2 = ||X||^2 + ||batch||^2.  The state
// (P, ||X||^2, valid) lives in the model buffer (checkpointed and restored with it).
// Every sum here is exact algebra of the same quantity the full pass computes; only the
// rounding order differs (fp32 runs of <= I / 32 products per lane, fp64 across).
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace sbt {

namespace {

constexpr int kFT = 512;            // threads per block (one block per SM: As fills the shared memory)
constexpr int kFW = kFT / 32;

// One row (j, k) of the store per warp; lane l takes the column quads l, l + 32, ... of the
// row (float4 loads; the store's padding columns are zero).  acc[f] += (sum over the lane's
// columns of X(i,j,k) As(i,f)) * w(j,k,f): the row weight multiplies the lane partial
// (linearity), so no reduction per row is needed.  As is staged transposed in shared memory,
// As_s[f][i] (padded to the pitch with zeros), so a lane reads its four columns of component f
// with one conflict-free 16-byte load.
template <int RB>
__global__ void __launch_bounds__(kFT) fitrows_kernel(FitRows a, double* __restrict__ part) {
  extern __shared__ __align__(16) float As_s[];
  const int R = a.R;
  int64_t nrows;
  if (a.gate && *a.gate != a.gate_val) nrows = 0;   // device-side plan (no host round trip)
  else if (a.kind == 0) nrows = (a.k1 - a.k0) * a.J;
  else {
    const int nl = *a.nlist;
    nrows = a.kind == 1 ? (int64_t)nl * (a.k1 - a.k0) : (int64_t)nl * a.J;
  }
  if (nrows <= (int64_t)blockIdx.x * kFW) {   // no row for this block: zero partials
    if (threadIdx.x < RB + 1) part[(int64_t)blockIdx.x * (RB + 1) + threadIdx.x] = 0.0;
    return;
  }
  const int P = (int)a.pitch;
  for (int e = threadIdx.x; e < R * P; e += blockDim.x) {
    const int f = e / P, i = e - f * P;
    As_s[e] = i < a.I ? a.As[(int64_t)i * R + f] : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nq = P / 4;
  double acc[RB + 1];
#pragma unroll
  for (int f = 0; f <= RB; ++f) acc[f] = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * kFW + warp; row < nrows; row += (int64_t)gridDim.x * kFW) {
    int64_t j, k;
    if (a.kind == 0) { k = a.k0 + row / a.J; j = row - (k - a.k0) * a.J; }
    else if (a.kind == 1) { const int64_t t = row / (a.k1 - a.k0); j = a.list[t]; k = a.k0 + (row - t * (a.k1 - a.k0)); }
    else { const int64_t t = row / a.J; j = row - t * a.J; k = a.list[t]; }
    const int64_t kg = a.kmap ? a.kmap[k] : k;   // store slice -> model row (sharded)
    const float4* x = reinterpret_cast<const float4*>(a.X + (k * a.J + j) * a.pitch);
    float d[RB];
#pragma unroll
    for (int f = 0; f < RB; ++f) d[f] = 0.f;
    float ss = 0.f;
    // four quads per step: four 16-byte loads in flight per lane before the arithmetic
    for (int q0 = lane; q0 < nq; q0 += 128) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + 32 * u;
        v[u] = q < nq ? __ldg(x + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + 32 * u;
        if (q >= nq) break;
        ss = fmaf(v[u].x, v[u].x, fmaf(v[u].y, v[u].y, fmaf(v[u].z, v[u].z, fmaf(v[u].w, v[u].w, ss))));
#pragma unroll
        for (int f = 0; f < RB; ++f) {
          if (f < R) {
            const float4 w = reinterpret_cast<const float4*>(As_s + f * P)[q];
            d[f] = fmaf(v[u].x, w.x, fmaf(v[u].y, w.y, fmaf(v[u].z, w.z, fmaf(v[u].w, w.w, d[f]))));
          }
        }
      }
    }
#pragma unroll
    for (int f = 0; f < RB; ++f) {
      if (f < R) {
        float u = a.U[j * R + f], v = a.V[kg * R + f];
        if (a.Usub) u -= a.Usub[j * R + f];
        if (a.Vsub) v -= a.Vsub[kg * R + f];
        acc[f] += (double)d[f] * ((double)u * (double)v);
      }
    }
    acc[RB] += (double)ss;
  }
  // block reduction (fixed order): warp butterflies, then over the warps
  __shared__ double red[kFW][RB + 1];
#pragma unroll
  for (int f = 0; f <= RB; ++f) {
    double v = acc[f];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][f] = v;
  }
  __syncthreads();
  if (threadIdx.x <= RB) {
    double s = 0.0;
    for (int w = 0; w < kFW; ++w) s += red[w][threadIdx.x];
    part[(int64_t)blockIdx.x * (RB + 1) + threadIdx.x] = s;
  }
}

// Plan of the incremental fit (one block, deterministic ordered compaction):
//   mode 1 (incremental) if the old state is valid, A' == A, and the changed B rows x old
//   slices + changed old C rows x J stay within `budget` rows; else mode 2 (full pass).
//   jlist / klist: the changed B rows / old C rows in increasing order.
__global__ void fitinc_plan_kernel(FitPlanArgs p) {
  __shared__ int s_cnt[2], s_anyA, s_base;
  __shared__ int s_scan[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) { s_anyA = 0; s_cnt[0] = s_cnt[1] = 0; }
  __syncthreads();
  // A unchanged?
  for (int64_t e = tid; e < (int64_t)p.I * p.R; e += nt)
    if (p.A1[e] != p.A0[e]) s_anyA = 1;
  // ordered compaction of changed rows of B (m = 0) and of the old rows of C (m = 1)
  for (int m = 0; m < 2; ++m) {
    const float* F1 = m == 0 ? p.B1 : p.C1;
    const float* F0 = m == 0 ? p.B0 : p.C0;
    const int64_t n = m == 0 ? p.J : p.Kold;
    int32_t* out = m == 0 ? p.jlist : p.klist;
    for (int64_t base = 0; base < n; base += nt) {
      const int64_t r = base + tid;
      int ch = 0;
      if (r < n)
        for (int f = 0; f < p.R; ++f) ch |= F1[r * p.R + f] != F0[r * p.R + f];
      s_scan[tid] = ch;
      __syncthreads();
      for (int o = 1; o < nt; o <<= 1) {   // inclusive Hillis-Steele scan
        const int v = tid >= o ? s_scan[tid - o] : 0;
        __syncthreads();
        s_scan[tid] += v;
        __syncthreads();
      }
      if (tid == 0) s_base = s_cnt[m];
      __syncthreads();
      if (ch) out[s_base + s_scan[tid] - 1] = (int32_t)r;
      __syncthreads();
      if (tid == nt - 1) s_cnt[m] += s_scan[nt - 1];
      __syncthreads();
    }
  }
  __syncthreads();
  if (tid == 0) {
    const bool valid = p.st_old[p.R + 1] == 1.0;
    const double rows = (double)s_cnt[0] * (double)p.Kold + (double)s_cnt[1] * (double)p.J;
    const int incr = valid && !s_anyA && rows <= p.budget_rows && (p.allow_c || s_cnt[1] == 0);
    *p.mode = incr ? 1 : 2;
    p.counts[0] = s_cnt[0];
    p.counts[1] = s_cnt[1];
  }
}

// Sum of the block partials of the terms the plan selected (terms 0..2: incremental; term 3:
// the full pass) into out[R + 1]: thread t < R + 1 sums column t over the terms and blocks in a
// fixed order with four independent chains (deterministic; no serial chain of 4 x blocks).
__device__ void fitinc_terms_sum(const FitFinishArgs& a, bool incr, double* out) {
  // thread t sums the blocks b = t, t + nt, ... of every selected term (a fixed assignment), then
  // each column is reduced across the threads by the fixed tree of block_sum_d: deterministic,
  // and the partials' loads are spread over the whole block (one thread per column serialised
  // ~1200 dependent L2 loads: ~100 us)
  __shared__ double red[32];
  const int R = a.R, RB = a.RB, t = threadIdx.x, nt = blockDim.x;
  double s[kMaxR + 1];
  for (int c = 0; c <= R; ++c) s[c] = 0.0;
  for (int tm = 0; tm < 4; ++tm) {
    const double* pt = a.terms[tm];
    if (!pt || incr != (tm < 3)) continue;
    const bool sq = !(tm == 1 || tm == 2);   // ||X||^2 grows by the new slices only
    for (int b = t; b < a.nparts[tm]; b += nt) {
      const double* row = pt + (int64_t)b * (RB + 1);
      for (int c = 0; c < R; ++c) s[c] += row[c];
      if (sq) s[R] += row[RB];
    }
  }
  for (int c = 0; c <= R; ++c) {
    const double v = block_sum_d(s[c], red);
    if (t == 0) out[c] = v;
  }
}

// P' (incremental: P + the selected terms; full: the full pass), ||X'||^2, the relative
// error from lam' and the Grams; writes the new state (valid).
__global__ void fitinc_finish_kernel(FitFinishArgs a) {
  __shared__ double sums[kMaxR + 1];
  const int R = a.R;
  const bool incr = *a.mode == 1;
  if (a.reduced) {
    if (threadIdx.x <= R) sums[threadIdx.x] = a.reduced[threadIdx.x];
  } else {
    fitinc_terms_sum(a, incr, sums);
  }
  __shared__ double Gs[3 * kMaxR * kMaxR], ls[kMaxR], so[kMaxR + 2];
  for (int e = threadIdx.x; e < 3 * R * R; e += blockDim.x) Gs[e] = a.G[e];   // staged: thread 0's
  for (int e = threadIdx.x; e < R; e += blockDim.x) ls[e] = (double)a.lam[e];  // loops read shared
  for (int e = threadIdx.x; e < R + 1; e += blockDim.x) so[e] = a.st_old[e];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double P[kMaxR];
  for (int f = 0; f < R; ++f) P[f] = (incr ? so[f] : 0.0) + sums[f];
  const double xsq = (incr ? so[R] : 0.0) + sums[R];
  double inner = 0.0, mn = 0.0;
  for (int f = 0; f < R; ++f) inner += ls[f] * P[f];
  for (int f = 0; f < R; ++f)
    for (int g = 0; g < R; ++g)
      mn += ls[f] * ls[g] * Gs[f * R + g] * Gs[R * R + f * R + g] * Gs[2 * R * R + f * R + g];
  const double res = fmax(0.0, xsq - 2.0 * inner + mn);
  *a.relerr = xsq > 0.0 ? sqrt(res / xsq) : 0.0;
  for (int f = 0; f < R; ++f) a.st_new[f] = P[f];
  a.st_new[R] = xsq;
  a.st_new[R + 1] = 1.0;
}

// the selected terms' sums into out[R + 1] (sharded: before the all-reduce)
__global__ void fitinc_sum_kernel(FitFinishArgs a, double* out) {
  fitinc_terms_sum(a, *a.mode == 1, out);
}

// COO: one thread per entry (grid-stride, fixed order per thread), the product of the three
// factor entries in fp32 (as the summary fits), each component's sum in fp64; block sums in the
// fixed tree order of block_sum_d
template <int RB>
__global__ void __launch_bounds__(256) coo_fitrows_kernel(CooFitRows a, double* __restrict__ part) {
  __shared__ double red[32];
  if (a.gate && *a.gate != a.gate_val) return;
  const int R = a.R;
  double acc[RB + 1];
#pragma unroll
  for (int f = 0; f <= RB; ++f) acc[f] = 0.0;
  if (a.bA) {   // the difference term over the old entries
    if (*a.any == 0) {   // no changed row: zero partials
      if (threadIdx.x <= RB) part[(int64_t)blockIdx.x * (RB + 1) + threadIdx.x] = 0.0;
      return;
    }
    for (int64_t e = a.n0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.n1;
         e += (int64_t)gridDim.x * blockDim.x) {
      const int i = a.i[e], j = a.j[e], k = a.k[e];
      if (!(((a.bA[i >> 5] >> (i & 31)) | (a.bB[j >> 5] >> (j & 31)) | (a.bC[k >> 5] >> (k & 31))) & 1u)) continue;
      const float v = a.v[e];
      const float *ra = a.A + (int64_t)i * R, *rb = a.B + (int64_t)j * R, *rc = a.C + (int64_t)k * R;
      const float *oa = a.A0 + (int64_t)i * R, *ob = a.B0 + (int64_t)j * R, *oc = a.C0 + (int64_t)k * R;
#pragma unroll
      for (int f = 0; f < RB; ++f)
        if (f < R) acc[f] += (double)v * ((double)(ra[f] * rb[f] * rc[f]) - (double)(oa[f] * ob[f] * oc[f]));
    }
  } else {
    for (int64_t e = a.n0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.n1;
         e += (int64_t)gridDim.x * blockDim.x) {
      const float v = a.v[e];
      const float* ra = a.A + (int64_t)a.i[e] * R;
      const float* rb = a.B + (int64_t)a.j[e] * R;
      const float* rc = a.C + (int64_t)a.k[e] * R;
#pragma unroll
      for (int f = 0; f < RB; ++f)
        if (f < R) acc[f] += (double)v * (double)(ra[f] * rb[f] * rc[f]);
      acc[RB] += (double)v * (double)v;
    }
  }
  for (int f = 0; f <= RB; ++f) {
    if (f < R || f == RB) {
      const double t = block_sum_d(acc[f], red);
      if (threadIdx.x == 0) part[(int64_t)blockIdx.x * (RB + 1) + f] = t;
    }
  }
}

// one thread per model row of A, B and the old rows of C: a row differing in any entry sets
// its bit (and *any); thread 0 writes the plan mode
__global__ void coo_fit_flags_kernel(CooFitFlags p) {
  const int64_t n = p.I + p.J + p.Kold;
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.mode = p.st_old[p.R + 1] == 1.0 ? 1 : 2;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const float *x0, *x1;
    uint32_t* bm;
    int64_t r;
    if (t < p.I) { r = t; x0 = p.A0; x1 = p.A1; bm = p.bA; }
    else if (t < p.I + p.J) { r = t - p.I; x0 = p.B0; x1 = p.B1; bm = p.bB; }
    else { r = t - p.I - p.J; x0 = p.C0; x1 = p.C1; bm = p.bC; }
    bool ch = false;
    for (int f = 0; f < p.R; ++f) ch |= x0[r * p.R + f] != x1[r * p.R + f];
    if (ch) {
      atomicOr(bm + (r >> 5), 1u << (r & 31));
      atomicOr(p.any, 1);
    }
  }
}

// Column-owner variant (RB <= 12): thread t of column block cb owns the column quad
// cb * 256 + t of every row and keeps As for its 4 columns in registers (4 RB floats), so the
// per-element work is R FFMAs with no shared-memory operand traffic; a block walks a contiguous
// range of rows in chunks of kCR, whose store offsets and weights w_f = U(j,f) V(k,f) (with the
// Usub / Vsub differences) are formed once per chunk in shared memory.  Row-chunk partials in
// fp32 (<= 16 rows), fp64 across; grid = fitrows_blocks(): nrg row groups x ncb column blocks
// (the blocks past ncb * nrg write zero partials).
constexpr int kCT2 = 256, kCR = 64, kRF = 8;   // kRF: rows whose 16-byte loads are in flight
template <int RB>
__global__ void __launch_bounds__(kCT2, 2) fitcols_kernel(FitRows a, double* __restrict__ part) {
  __shared__ float Wsh[kCR][RB];
  __shared__ int64_t Xoff[kCR];
  __shared__ double red[32];
  const int R = a.R, tid = threadIdx.x;
  const int nq = (int)(a.pitch / 4), ncb = (nq + kCT2 - 1) / kCT2;
  const int nrg = (int)gridDim.x / ncb;
  const int cb = blockIdx.x % ncb, rg = blockIdx.x / ncb;
  int64_t nrows;
  if (a.gate && *a.gate != a.gate_val) nrows = 0;
  else if (a.kind == 0) nrows = (a.k1 - a.k0) * a.J;
  else {
    const int nl = *a.nlist;
    nrows = a.kind == 1 ? (int64_t)nl * (a.k1 - a.k0) : (int64_t)nl * a.J;
  }
  const int64_t per = nrg > 0 ? (nrows + nrg - 1) / nrg : 0;
  const int64_t r0 = (int64_t)rg * per, r1 = min(nrows, r0 + per);
  if (rg >= nrg || r0 >= r1) {
    if (tid <= RB) part[(int64_t)blockIdx.x * (RB + 1) + tid] = 0.0;
    return;
  }
  const int q = cb * kCT2 + tid;
  const bool valid = q < nq;
  float av[RB][4];
#pragma unroll
  for (int f = 0; f < RB; ++f)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * q + e;
      av[f][e] = (valid && f < R && i < a.I) ? a.As[(int64_t)i * R + f] : 0.f;
    }
  double acc[RB + 1];
#pragma unroll
  for (int f = 0; f <= RB; ++f) acc[f] = 0.0;
  for (int64_t c0 = r0; c0 < r1; c0 += kCR) {
    const int nrc = (int)min((int64_t)kCR, r1 - c0);
    __syncthreads();   // the previous chunk's offsets / weights are consumed
    if (tid < nrc) {
      const int64_t row = c0 + tid;
      int64_t j, k;
      if (a.kind == 0) { k = a.k0 + row / a.J; j = row - (k - a.k0) * a.J; }
      else if (a.kind == 1) { const int64_t t = row / (a.k1 - a.k0); j = a.list[t]; k = a.k0 + (row - t * (a.k1 - a.k0)); }
      else { const int64_t t = row / a.J; j = row - t * a.J; k = a.list[t]; }
      const int64_t kg = a.kmap ? a.kmap[k] : k;   // store slice -> model row (sharded)
      Xoff[tid] = (k * a.J + j) * a.pitch;
#pragma unroll
      for (int f = 0; f < RB; ++f) {
        float w = 0.f;
        if (f < R) {
          float u = a.U[j * R + f], v = a.V[kg * R + f];
          if (a.Usub) u -= a.Usub[j * R + f];
          if (a.Vsub) v -= a.Vsub[kg * R + f];
          w = u * v;
        }
        Wsh[tid][f] = w;
      }
    }
    __syncthreads();
    if (!valid) continue;
    for (int rb = 0; rb < nrc; rb += 16) {
      float accf[RB];
#pragma unroll
      for (int f = 0; f < RB; ++f) accf[f] = 0.f;
      float ss = 0.f;
      const int re = min(nrc, rb + 16);
      for (int rr = rb; rr < re; rr += kRF) {
        float4 x[kRF];
#pragma unroll
        for (int u = 0; u < kRF; ++u)   // kRF rows' loads in flight
          x[u] = rr + u < re ? __ldg(reinterpret_cast<const float4*>(a.X + Xoff[rr + u]) + q)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < kRF; ++u) {
          if (rr + u >= re) break;
          ss = fmaf(x[u].x, x[u].x, fmaf(x[u].y, x[u].y, fmaf(x[u].z, x[u].z, fmaf(x[u].w, x[u].w, ss))));
#pragma unroll
          for (int f = 0; f < RB; ++f) {
            const float d = fmaf(x[u].x, av[f][0], fmaf(x[u].y, av[f][1], fmaf(x[u].z, av[f][2], x[u].w * av[f][3])));
            accf[f] = fmaf(d, Wsh[rr + u][f], accf[f]);
          }
        }
      }
#pragma unroll
      for (int f = 0; f < RB; ++f) acc[f] += (double)accf[f];
      acc[RB] += (double)ss;
    }
  }
#pragma unroll
  for (int f = 0; f <= RB; ++f) {
    const double t = block_sum_d(acc[f], red);
    if (tid == 0) part[(int64_t)blockIdx.x * (RB + 1) + f] = t;
  }
}

template <int RB>
cudaError_t fitrows_rb(const FitRows& a, double* part, int nblocks, cudaStream_t st) {
  if (RB <= 12 && !getenv("SAMBATEN_FITROWS_SMEM")) {
    fitcols_kernel<RB <= 12 ? RB : 12><<<nblocks, kCT2, 0, st>>>(a, part);
    return cudaGetLastError();
  }
  const size_t smem = sizeof(float) * (size_t)a.pitch * a.R;
  cudaFuncSetAttribute(fitrows_kernel<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fitrows_kernel<RB><<<nblocks, kFT, smem, st>>>(a, part);
  return cudaGetLastError();
}

}  // namespace

int fitrows_rb_of(int R) { return R <= 4 ? 4 : R <= 8 ? 8 : R <= 10 ? 10 : R <= 12 ? 12 : R <= 16 ? 16 : 32; }

int fitrows_blocks() { return kNumSMs * 2; }

bool fitrows_supported(int64_t pitch, int R) {
  return pitch % 4 == 0 && (size_t)pitch * R * sizeof(float) <= 200 * 1024;
}

cudaError_t launch_fitrows(FitRows a, double* part, cudaStream_t st) {
  if (!fitrows_supported(a.pitch, a.R)) return cudaErrorInvalidValue;
  const int nb = fitrows_blocks();
  switch (fitrows_rb_of(a.R)) {
    case 4: return fitrows_rb<4>(a, part, nb, st);
    case 8: return fitrows_rb<8>(a, part, nb, st);
    case 10: return fitrows_rb<10>(a, part, nb, st);
    case 12: return fitrows_rb<12>(a, part, nb, st);
    case 16: return fitrows_rb<16>(a, part, nb, st);
    default: return fitrows_rb<32>(a, part, nb, st);
  }
}

cudaError_t launch_coo_fitrows(const CooFitRows& a, double* part, cudaStream_t st) {
  const int nb = fitrows_blocks();
  switch (fitrows_rb_of(a.R)) {
    case 4: coo_fitrows_kernel<4><<<nb, 256, 0, st>>>(a, part); break;
    case 8: coo_fitrows_kernel<8><<<nb, 256, 0, st>>>(a, part); break;
    case 10: coo_fitrows_kernel<10><<<nb, 256, 0, st>>>(a, part); break;
    case 12: coo_fitrows_kernel<12><<<nb, 256, 0, st>>>(a, part); break;
    case 16: coo_fitrows_kernel<16><<<nb, 256, 0, st>>>(a, part); break;
    default: coo_fitrows_kernel<32><<<nb, 256, 0, st>>>(a, part); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_coo_fit_flags(const CooFitFlags& f, cudaStream_t st) {
  const int64_t n = f.I + f.J + f.Kold;
  const unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), kNumSMs * 8));
  coo_fit_flags_kernel<<<nb, 256, 0, st>>>(f);
  return cudaGetLastError();
}

cudaError_t launch_fitinc_plan(const FitPlanArgs& p, cudaStream_t st) {
  fitinc_plan_kernel<<<1, 1024, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fitinc_finish(const FitFinishArgs& a, cudaStream_t st) {
  fitinc_finish_kernel<<<1, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fitinc_sum(const FitFinishArgs& a, double* out, cudaStream_t st) {
  fitinc_sum_kernel<<<1, 256, 0, st>>>(a, out);
  return cudaGetLastError();
}

}  // namespace sbt
