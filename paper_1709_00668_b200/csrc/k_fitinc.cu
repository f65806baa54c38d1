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
#include "common.cuh"
#include "internal.h"

namespace sbt {

namespace {

constexpr int kFT = 256;            // threads per block
constexpr int kFW = kFT / 32;

// One row (j, k) of the store per warp; lane l takes the columns l, l + 32, ... of the row.
// acc[f] += (sum over the lane's columns of X(i,j,k) As(i,f)) * w(j,k,f): the row weight
// multiplies the lane partial (linearity), so no reduction per row is needed.  As (I x R)
// is staged in shared memory when it fits, else read through L1.
template <int RB>
__global__ void __launch_bounds__(kFT) fitrows_kernel(FitRows a, double* __restrict__ part) {
  extern __shared__ __align__(16) float As_s[];
  const int R = a.R;
  if (a.gate && *a.gate != a.gate_val) {   // device-side plan (no host round trip)
    if (threadIdx.x < RB + 1) part[(int64_t)blockIdx.x * (RB + 1) + threadIdx.x] = 0.0;
    return;
  }
  const bool smem_as = a.as_in_smem;
  if (smem_as) {
    for (int e = threadIdx.x; e < a.I * R; e += blockDim.x) As_s[e] = a.As[e];
    __syncthreads();
  }
  const float* As = smem_as ? As_s : a.As;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t nrows;
  int nl = 0;
  if (a.kind == 0) nrows = (a.k1 - a.k0) * a.J;
  else {
    nl = *a.nlist;
    nrows = a.kind == 1 ? (int64_t)nl * (a.k1 - a.k0) : (int64_t)nl * a.J;
  }
  double acc[RB + 1];
#pragma unroll
  for (int f = 0; f <= RB; ++f) acc[f] = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * kFW + warp; row < nrows; row += (int64_t)gridDim.x * kFW) {
    int64_t j, k;
    if (a.kind == 0) { k = a.k0 + row / a.J; j = row - (k - a.k0) * a.J; }
    else if (a.kind == 1) { const int64_t t = row / (a.k1 - a.k0); j = a.list[t]; k = a.k0 + (row - t * (a.k1 - a.k0)); }
    else { const int64_t t = row / a.J; j = row - t * a.J; k = a.list[t]; }
    // k is a slice of the store: local (sharded) -> model row through kmap; kind 2 lists hold
    // store slices too (the caller maps)
    const int64_t kg = a.kmap ? a.kmap[k] : k;
    const float* x = a.X + (k * a.J + j) * a.pitch;
    float d[RB];
#pragma unroll
    for (int f = 0; f < RB; ++f) d[f] = 0.f;
    float ss = 0.f;
    for (int i = lane; i < a.I; i += 32) {
      const float v = x[i];
      ss = fmaf(v, v, ss);
      const float* ar = As + (int64_t)i * R;
#pragma unroll
      for (int f = 0; f < RB; ++f)
        if (f < R) d[f] = fmaf(v, ar[f], d[f]);
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
  // block reduction (fixed order): warp butterflies, then warp 0 over the warps
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

// P' (incremental: P + the three term partials; full: the full pass's partials), ||X'||^2,
// the relative error from lam' and the Grams; writes the new state (valid).
__global__ void fitinc_finish_kernel(FitFinishArgs a) {
  if (threadIdx.x != 0) return;
  const int R = a.R, RB = a.RB;
  const bool incr = *a.mode == 1;
  double P[kMaxR];
  double xsq;
  for (int f = 0; f < R; ++f) P[f] = incr ? a.st_old[f] : 0.0;
  xsq = incr ? a.st_old[R] : 0.0;
  for (int t = 0; t < 4; ++t) {
    const double* pt = a.terms[t];
    if (!pt) continue;
    if (incr != (t < 3)) continue;   // terms 0..2: incremental; term 3: full pass
    for (int b = 0; b < a.nparts[t]; ++b) {
      for (int f = 0; f < R; ++f) P[f] += pt[(int64_t)b * (RB + 1) + f];
      if (t == 0 || t == 3) xsq += pt[(int64_t)b * (RB + 1) + RB];   // ||batch||^2 / ||X'||^2
    }
  }
  if (a.reduced) {   // sharded: the per-rank sums were all-reduced into reduced[R + 1]
    for (int f = 0; f < R; ++f) P[f] = (incr ? a.st_old[f] : 0.0) + a.reduced[f];
    xsq = (incr ? a.st_old[R] : 0.0) + a.reduced[R];
  }
  double inner = 0.0, mn = 0.0;
  for (int f = 0; f < R; ++f) inner += (double)a.lam[f] * P[f];
  for (int f = 0; f < R; ++f)
    for (int g = 0; g < R; ++g)
      mn += (double)a.lam[f] * (double)a.lam[g] * a.G[f * R + g] * a.G[R * R + f * R + g] * a.G[2 * R * R + f * R + g];
  const double res = fmax(0.0, xsq - 2.0 * inner + mn);
  *a.relerr = xsq > 0.0 ? sqrt(res / xsq) : 0.0;
  for (int f = 0; f < R; ++f) a.st_new[f] = P[f];
  a.st_new[R] = xsq;
  a.st_new[R + 1] = 1.0;
}

// sum of the block partials of every term into out[R + 1] (sharded: before the all-reduce)
__global__ void fitinc_sum_kernel(FitFinishArgs a, double* out) {
  if (threadIdx.x != 0) return;
  const int R = a.R, RB = a.RB;
  const bool incr = *a.mode == 1;
  for (int f = 0; f <= R; ++f) out[f] = 0.0;
  for (int t = 0; t < 4; ++t) {
    const double* pt = a.terms[t];
    if (!pt || incr != (t < 3)) continue;
    for (int b = 0; b < a.nparts[t]; ++b) {
      for (int f = 0; f < R; ++f) out[f] += pt[(int64_t)b * (RB + 1) + f];
      if (t == 0 || t == 3) out[R] += pt[(int64_t)b * (RB + 1) + RB];
    }
  }
}

template <int RB>
cudaError_t fitrows_rb(const FitRows& a, double* part, int nblocks, cudaStream_t st) {
  size_t smem = a.as_in_smem ? sizeof(float) * (size_t)a.I * a.R : 0;
  cudaFuncSetAttribute(fitrows_kernel<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fitrows_kernel<RB><<<nblocks, kFT, smem, st>>>(a, part);
  return cudaGetLastError();
}

}  // namespace

int fitrows_rb_of(int R) { return R <= 4 ? 4 : R <= 8 ? 8 : R <= 12 ? 12 : R <= 16 ? 16 : 32; }

int fitrows_blocks() { return kNumSMs * 4; }

cudaError_t launch_fitrows(FitRows a, double* part, cudaStream_t st) {
  a.as_in_smem = (size_t)a.I * a.R * sizeof(float) <= 160 * 1024;
  const int nb = fitrows_blocks();
  switch (fitrows_rb_of(a.R)) {
    case 4: return fitrows_rb<4>(a, part, nb, st);
    case 8: return fitrows_rb<8>(a, part, nb, st);
    case 12: return fitrows_rb<12>(a, part, nb, st);
    case 16: return fitrows_rb<16>(a, part, nb, st);
    default: return fitrows_rb<32>(a, part, nb, st);
  }
}

cudaError_t launch_fitinc_plan(const FitPlanArgs& p, cudaStream_t st) {
  fitinc_plan_kernel<<<1, 1024, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fitinc_finish(const FitFinishArgs& a, cudaStream_t st) {
  fitinc_finish_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fitinc_sum(const FitFinishArgs& a, double* out, cudaStream_t st) {
  fitinc_sum_kernel<<<1, 32, 0, st>>>(a, out);
  return cudaGetLastError();
}

}  // namespace sbt
