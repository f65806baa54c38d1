// k_fit.cu -- a7: relative error ||X - [[lam; A, B, C]]||_F / ||X||_F (R21).
//
// ||X - M||^2 = ||X||^2 - 2 <X, M> + ||M||^2 with <X, M> = sum_{j,k} sum_f d_f(j,k) lam_f
// B(j,f) C(k,f), d_f(j,k) = sum_i X(i,j,k) A(i,f), and ||M||^2 = lam^T (A^T A * B^T B * C^T C)
// lam.  One streaming pass over X (warp per 32 rows, 32 x 32 shared-memory tiles as in the
// ALS D-pass); fp64 partials per block, reduced in a fixed order.
#include "common.cuh"
#include "internal.h"

namespace sbt {

constexpr int kFitThreads = 256;

template <int RB>
__global__ void __launch_bounds__(kFitThreads) fit_pass_kernel(
    const float* __restrict__ X, int64_t I, int64_t J, int64_t pitch, int64_t nrows,
    const float* __restrict__ lam, const float* __restrict__ A, const float* __restrict__ B,
    const float* __restrict__ C, int R, int rows_per_block, double* part) {
  constexpr int S4 = (RB + 3) & ~3;
  constexpr int NW = RB <= 12 ? 8 : 4;
  __shared__ float tile_sh[NW][32][33];
  __shared__ __align__(16) float uc_sh[NW][32 * S4];
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float (*tile)[33] = tile_sh[warp];
  float* uc = uc_sh[warp];
  double inner = 0.0, sq = 0.0;
  const int64_t rb = (int64_t)blockIdx.x * rows_per_block;
  const int64_t re = min(rb + (int64_t)rows_per_block, nrows);
  for (int64_t row0 = rb + warp * 32; row0 < re; row0 += NW * 32) {
    const int nr = (int)min((int64_t)32, re - row0);
    float acc[RB];
    double acc64[RB];
#pragma unroll
    for (int f = 0; f < RB; ++f) { acc[f] = 0.f; acc64[f] = 0.0; }
    for (int pc = 0; pc < I; pc += 32) {
      const int w = (int)min((int64_t)32, I - pc);
#pragma unroll 8
      for (int r2 = 0; r2 < 32; ++r2)
        tile[r2][lane] = (r2 < nr && lane < w) ? __ldcs(X + (row0 + r2) * pitch + pc + lane) : 0.f;
#pragma unroll
      for (int f = 0; f < S4; ++f)
        uc[lane * S4 + f] = (lane < w && f < R) ? A[(int64_t)(pc + lane) * R + f] : 0.f;
      __syncwarp();
      for (int pp = 0; pp < w; ++pp) {
        const float y = tile[lane][pp];
        sq += (double)y * (double)y;
        const float4* u4 = reinterpret_cast<const float4*>(uc + pp * S4);
#pragma unroll
        for (int f4 = 0; f4 < S4 / 4; ++f4) {
          const float4 u = u4[f4];
          if (4 * f4 + 0 < RB) acc[4 * f4 + 0] = fmaf(y, u.x, acc[4 * f4 + 0]);
          if (4 * f4 + 1 < RB) acc[4 * f4 + 1] = fmaf(y, u.y, acc[4 * f4 + 1]);
          if (4 * f4 + 2 < RB) acc[4 * f4 + 2] = fmaf(y, u.z, acc[4 * f4 + 2]);
          if (4 * f4 + 3 < RB) acc[4 * f4 + 3] = fmaf(y, u.w, acc[4 * f4 + 3]);
        }
      }
#pragma unroll
      for (int f = 0; f < RB; ++f) { acc64[f] += (double)acc[f]; acc[f] = 0.f; }
      __syncwarp();
    }
    if (lane < nr) {
      const int64_t gr = row0 + lane;
      const int64_t k = gr / J, j = gr - k * J;
#pragma unroll
      for (int f = 0; f < RB; ++f)
        if (f < R)
          inner += acc64[f] * (double)lam[f] * (double)B[j * R + f] * (double)C[k * R + f];
    }
  }
  inner = block_sum_d(inner, red);
  sq = block_sum_d(sq, red);
  if (threadIdx.x == 0) {
    part[2 * (int64_t)blockIdx.x] = inner;
    part[2 * (int64_t)blockIdx.x + 1] = sq;
  }
}

__device__ double gram_entry(const float* U, int64_t n, int R, int f, int g) {
  double s = 0.0;
  for (int64_t row = 0; row < n; ++row) s += (double)U[row * R + f] * (double)U[row * R + g];
  return s;
}

__global__ void fit_final_kernel(const double* part, int nb, const float* lam, const float* A,
                                 const float* B, const float* C, int64_t I, int64_t J,
                                 int64_t K, int R, double* relerr) {
  __shared__ double Mn[kMaxR * kMaxR];
  for (int pr = threadIdx.x; pr < R * R; pr += blockDim.x) {
    const int f = pr / R, g = pr - f * R;
    Mn[pr] = (double)lam[f] * (double)lam[g] * gram_entry(A, I, R, f, g) *
             gram_entry(B, J, R, f, g) * gram_entry(C, K, R, f, g);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double inner = 0.0, sq = 0.0, mn = 0.0;
    for (int b = 0; b < nb; ++b) { inner += part[2 * b]; sq += part[2 * b + 1]; }
    for (int pr = 0; pr < R * R; ++pr) mn += Mn[pr];
    const double res = fmax(0.0, sq - 2.0 * inner + mn);
    *relerr = sq > 0.0 ? sqrt(res / sq) : 0.0;
  }
}

static int fit_blocks(const DenseView& X) {
  const int64_t nrows = X.J * X.K;
  int64_t nb = ceil_div(nrows, 256);
  if (nb > kNumSMs * 4) nb = kNumSMs * 4;
  if (nb < 1) nb = 1;
  return (int)nb;
}

size_t fit_dense_ws_doubles(const DenseView& X) { return 2 * (size_t)fit_blocks(X) + 8; }

template <int RB>
static cudaError_t fit_rb(const DenseView& X, const float* lam, const float* A, const float* B,
                          const float* C, int R, double* ws, double* relerr, cudaStream_t st) {
  const int64_t nrows = X.J * X.K;
  const int nb = fit_blocks(X);
  const int rpb = (int)ceil_div(nrows, nb);
  constexpr int NW = RB <= 12 ? 8 : 4;
  fit_pass_kernel<RB><<<nb, 32 * NW, 0, st>>>(X.base, X.I, X.J, X.pitch, nrows, lam, A, B, C,
                                                  R, rpb, ws);
  fit_final_kernel<<<1, 256, 0, st>>>(ws, nb, lam, A, B, C, X.I, X.J, X.K, R, relerr);
  return cudaGetLastError();
}

cudaError_t launch_fit_dense(const DenseView& X, const float* lam, const float* A,
                             const float* B, const float* C, int R, double* ws, double* relerr,
                             cudaStream_t st) {
  if (R <= 4) return fit_rb<4>(X, lam, A, B, C, R, ws, relerr, st);
  if (R <= 8) return fit_rb<8>(X, lam, A, B, C, R, ws, relerr, st);
  if (R <= 10) return fit_rb<10>(X, lam, A, B, C, R, ws, relerr, st);
  if (R <= 12) return fit_rb<12>(X, lam, A, B, C, R, ws, relerr, st);
  if (R <= 16) return fit_rb<16>(X, lam, A, B, C, R, ws, relerr, st);
  if (R <= 24) return fit_rb<24>(X, lam, A, B, C, R, ws, relerr, st);
  return fit_rb<32>(X, lam, A, B, C, R, ws, relerr, st);
}

}  // namespace sbt
