// k_als_rows.cu -- row-parallel R x R solve / normalise / Gram / fit of the batched ALS
// (Alg. 1 l.5 P:213; R10-R12), used by the COO summaries (large mode sizes: a single
// block per repetition would serialise thousands of rows).  Per mode m, after the MTTKRP
// has produced M (fp64 [rep][rows][R]):
//   als_vinv_kernel   (rep)          Vi = (*_{o != m} G_o)^-1: warp Gauss-Jordan, pinv fallback
//   als_rows_kernel   (row tile, rep) x = M Vi (fp64), partial Gram sum x x^T and, for mode 2,
//                                     partial fit inner product sum x M, per 256-row tile
//   als_reduce_kernel (rep)          tiles summed in order -> lambda (column norms), the
//                                     normalised Gram, and for mode 2 the fit / stop test
//   als_scale_kernel  (row tile, rep) U = fp32(x / lambda)
// The sums are over fixed tiles in a fixed order: deterministic.
#include "als_small.cuh"
#include "common.cuh"
#include "internal.h"

namespace sbt {

namespace {

constexpr int kRT = 128;   // rows per tile / threads per block

__global__ void als_vinv_kernel(RowsAls a, int mode) {
  const int rep = blockIdx.x;
  if (a.done[rep]) return;
  const int R = a.R, lane = threadIdx.x;
  __shared__ double V[kMaxR * kMaxR], W[2 * kMaxR * kMaxR], Q[kMaxR * kMaxR], fc[kMaxR];
  const double* G = a.G + (int64_t)rep * 3 * R * R;
  const int o1 = mode == 0 ? 1 : 0, o2 = mode == 2 ? 1 : 2;
  for (int idx = lane; idx < R * R; idx += 32) V[idx] = G[o1 * R * R + idx] * G[o2 * R * R + idx];
  __syncwarp();
  if (R <= 16) {
    bool ok = R <= 4 ? gj_reg<4>(V, a.Vi + (int64_t)rep * R * R, R)
            : R <= 8 ? gj_reg<8>(V, a.Vi + (int64_t)rep * R * R, R)
            : R <= 12 ? gj_reg<12>(V, a.Vi + (int64_t)rep * R * R, R)
                      : gj_reg<16>(V, a.Vi + (int64_t)rep * R * R, R);
    if (!ok && lane == 0) {
      pinv_R(V, a.Vi + (int64_t)rep * R * R, R, W, Q);
      a.flags[rep] |= 1;
    }
    return;
  }
  // Gauss-Jordan on [V | I] in shared memory (SPD: every pivot positive)
  const int Wd = 2 * R;
  for (int e = lane; e < R * Wd; e += 32) {
    const int i = e / Wd, c = e - i * Wd;
    W[e] = c < R ? V[i * R + c] : (c - R == i ? 1.0 : 0.0);
  }
  __syncwarp();
  bool ok = true;
  for (int j = 0; j < R; ++j) {
    const double piv = W[j * Wd + j];
    if (!(piv > 0.0)) { ok = false; break; }
    for (int i = lane; i < R; i += 32) fc[i] = W[i * Wd + j];
    __syncwarp();
    const double rp = 1.0 / piv;
    for (int c = lane; c < Wd; c += 32) W[j * Wd + c] *= rp;
    __syncwarp();
    for (int e = lane; e < R * Wd; e += 32) {
      const int i = e / Wd, c = e - i * Wd;
      if (i != j) W[e] -= fc[i] * W[j * Wd + c];
    }
    __syncwarp();
  }
  double* Vi = a.Vi + (int64_t)rep * R * R;
  if (ok) {
    for (int e = lane; e < R * R; e += 32) Vi[e] = W[(e / R) * Wd + R + (e % R)];
  } else if (lane == 0) {
    pinv_R(V, Vi, R, W, Q);
    a.flags[rep] |= 1;
  }
}

template <int RB>
__global__ void __launch_bounds__(kRT) als_rows_kernel(RowsAls a, int mode) {
  const int tile = blockIdx.x, rep = blockIdx.y;
  if (a.done[rep]) return;
  const int R = a.R;
  const int n = mode == 0 ? a.nI : mode == 1 ? a.nJ : a.nK;
  __shared__ double Vs[RB * RB];
  __shared__ double xs[kRT][RB + 1];
  __shared__ double ms[kRT][RB + 1];
  const double* Vi = a.Vi + (int64_t)rep * R * R;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Vs[e] = Vi[e];
  __syncthreads();
  const int row = tile * kRT + threadIdx.x;
  const double* M = a.M[mode] + rep * a.m_stride[mode];
  double* X = a.X + (int64_t)rep * a.x_stride;
  double m[RB], x[RB];
#pragma unroll
  for (int f = 0; f < RB; ++f) m[f] = (row < n && f < R) ? M[(int64_t)row * R + f] : 0.0;
#pragma unroll
  for (int f = 0; f < RB; ++f) {
    double s = 0.0;
#pragma unroll
    for (int g = 0; g < RB; ++g)
      if (g < R && f < R) s += m[g] * Vs[g * R + f];
    x[f] = s;
  }
#pragma unroll
  for (int f = 0; f < RB; ++f) {
    if (row < n && f < R) X[(int64_t)row * R + f] = x[f];
    xs[threadIdx.x][f] = x[f];
    ms[threadIdx.x][f] = m[f];
  }
  __syncthreads();
  // partial Gram of x over the tile (thread per (f, g) pair, rows in order) and fit inner
  const int ntile = (n + kRT - 1) / kRT;
  const int npair = R * R;
  double* part = a.part + ((int64_t)rep * ntile + tile) * (npair + 1);
  const int nr = min(kRT, n - tile * kRT);
  for (int pr = threadIdx.x; pr <= npair; pr += blockDim.x) {
    double s = 0.0;
    if (pr < npair) {
      const int f = pr / R, g = pr - f * R;
      for (int t = 0; t < nr; ++t) s += xs[t][f] * xs[t][g];
    } else if (mode == 2) {
      for (int t = 0; t < nr; ++t)
        for (int f = 0; f < R; ++f) s += xs[t][f] * ms[t][f];
    }
    part[pr] = s;
  }
}

__global__ void als_reduce_kernel(RowsAls a, int mode) {
  const int rep = blockIdx.x;
  if (a.done[rep]) return;
  const int R = a.R;
  const int n = mode == 0 ? a.nI : mode == 1 ? a.nJ : a.nK;
  const int ntile = (n + kRT - 1) / kRT;
  const int npair = R * R;
  __shared__ double Gx[kMaxR * kMaxR + 1];
  __shared__ double lam[kMaxR];
  const double* part = a.part + (int64_t)rep * ntile * (npair + 1);
  for (int pr = threadIdx.x; pr <= npair; pr += blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;   // 4 interleaved chains, fixed order
    int t = 0;
    for (; t + 3 < ntile; t += 4) {
      s0 += part[(int64_t)t * (npair + 1) + pr];
      s1 += part[(int64_t)(t + 1) * (npair + 1) + pr];
      s2 += part[(int64_t)(t + 2) * (npair + 1) + pr];
      s3 += part[(int64_t)(t + 3) * (npair + 1) + pr];
    }
    for (; t < ntile; ++t) s0 += part[(int64_t)t * (npair + 1) + pr];
    Gx[pr] = (s0 + s1) + (s2 + s3);
  }
  __syncthreads();
  if (threadIdx.x < R) {
    const double l = sqrt(Gx[threadIdx.x * R + threadIdx.x]);
    lam[threadIdx.x] = l;
    a.lam[rep * R + threadIdx.x] = l;
  }
  __syncthreads();
  double* G = a.G + (int64_t)rep * 3 * R * R + mode * R * R;
  for (int pr = threadIdx.x; pr < npair; pr += blockDim.x) {
    const int f = pr / R, g = pr - f * R;
    const double lf = lam[f] > 0.0 ? lam[f] : 1.0, lg = lam[g] > 0.0 ? lam[g] : 1.0;
    G[pr] = Gx[pr] / (lf * lg);
  }
  __syncthreads();
  __shared__ double G0[3 * kMaxR * kMaxR];   // the three Grams, staged for thread 0's sum
  if (mode == 2)
    for (int e = threadIdx.x; e < 3 * npair; e += blockDim.x) G0[e] = a.G[(int64_t)rep * 3 * npair + e];
  __syncthreads();
  if (mode == 2 && threadIdx.x == 0) {
    // fit = 1 - sqrt(||Y||^2 - 2 <Y, M> + ||M||^2) / ||Y||  with <Y, M> = sum x M2 (lambda
    // cancels) and ||M||^2 = lam^T (G0 * G1 * G2) lam
    double mn = 0.0;
    for (int f = 0; f < R; ++f)
      for (int g = 0; g < R; ++g)
        mn += lam[f] * lam[g] * G0[f * R + g] * G0[R * R + f * R + g] * G0[2 * R * R + f * R + g];
    const double inner = Gx[npair];
    const double y2 = a.ysq[rep];
    const double res = fmax(0.0, y2 - 2.0 * inner + mn);
    const double fit = y2 > 0.0 ? 1.0 - sqrt(res) / sqrt(y2) : 0.0;
    const int it = a.iters[rep] + 1;
    a.iters[rep] = it;
    const double prev = a.fit[rep];
    a.fit_prev[rep] = prev;
    a.fit[rep] = fit;
    bool stop = it >= a.maxit;
    if (it >= 2 && fabs(fit - prev) < a.tol) stop = true;
    if (!isfinite(fit)) { a.flags[rep] |= 2; stop = true; }
    a.stop[rep] = stop ? 1 : 0;
  }
}

__global__ void als_scale_kernel(RowsAls a, int mode) {
  const int tile = blockIdx.x, rep = blockIdx.y;
  if (a.done[rep]) return;
  const int R = a.R;
  const int n = mode == 0 ? a.nI : mode == 1 ? a.nJ : a.nK;
  const double* lam = a.lam + rep * R;
  const double* X = a.X + (int64_t)rep * a.x_stride;
  float* U = a.U[mode] + rep * a.u_stride[mode];
  const int row0 = tile * kRT;
  const int nel = (min(row0 + kRT, n) - row0) * R;   // the tile's elements (32-bit index math)
  float* Up = a.Up[mode] ? a.Up[mode] + rep * a.up_stride[mode] : nullptr;
  for (int e = threadIdx.x; e < nel; e += blockDim.x) {
    const int rl = e / R, f = e - rl * R;
    const int64_t t = (int64_t)row0 * R + e;
    const double l = lam[f];
    const float u = __double2float_rn(l > 0.0 ? X[t] / l : X[t]);
    U[t] = u;
    if (Up) Up[(int64_t)(row0 + rl) * a.RBp + f] = u;
  }
}

__global__ void pad_factors_kernel(RowsAls a) {
  const int m = blockIdx.y, rep = blockIdx.z;
  const int n = m == 0 ? a.nI : m == 1 ? a.nJ : a.nK;
  const float* U = a.U[m] + rep * a.u_stride[m];
  float* Up = a.Up[m] + rep * a.up_stride[m];
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * a.RBp;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / a.RBp;
    const int f = (int)(t - row * a.RBp);
    Up[t] = f < a.R ? U[row * a.R + f] : 0.f;
  }
}

// start of an iteration: a repetition whose last fit met the stop test is done
__global__ void als_commit_stop_kernel(RowsAls a) {
  const int rep = threadIdx.x;
  if (rep < a.r && a.stop[rep]) a.done[rep] = 1;
}

// ---------------------------------------------------------------------------------------
// Grams of up to 3 factors x r repetitions: tile partials (fp64, rows in order) + ordered
// combination.  G[rep][m][R][R] = U_m^T U_m.
// ---------------------------------------------------------------------------------------
__global__ void gram_tiles_kernel(GramArgs g) {
  const int tile = blockIdx.x, m = blockIdx.y, rep = blockIdx.z;
  const int R = g.R, n = g.n[m];
  const int tiles = (n + kRT - 1) / kRT;
  if (tile >= tiles) return;
  __shared__ float rows[kRT * kMaxR];
  const float* U = g.U[m] + rep * g.u_stride[m];
  const int r0 = tile * kRT, nr = min(kRT, n - r0);
  for (int e = threadIdx.x; e < nr * R; e += blockDim.x) rows[e] = U[(int64_t)r0 * R + e];
  __syncthreads();
  double* part = g.part + (((int64_t)rep * 3 + m) * g.tmax + tile) * R * R;
  for (int pr = threadIdx.x; pr < R * R; pr += blockDim.x) {
    const int f = pr / R, h = pr - f * R;
    double s = 0.0;
    for (int t = 0; t < nr; ++t) s += (double)rows[t * R + f] * (double)rows[t * R + h];
    part[pr] = s;
  }
}

__global__ void gram_combine_kernel(GramArgs g) {
  const int m = blockIdx.x, rep = blockIdx.y;
  const int R = g.R, n = g.n[m];
  const int tiles = (n + kRT - 1) / kRT;
  const double* part = g.part + ((int64_t)rep * 3 + m) * g.tmax * R * R;
  double* G = g.G + rep * g.g_stride + (int64_t)m * R * R;
  for (int pr = threadIdx.x; pr < R * R; pr += blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int t = 0;
    for (; t + 3 < tiles; t += 4) {
      s0 += part[(int64_t)t * R * R + pr];
      s1 += part[(int64_t)(t + 1) * R * R + pr];
      s2 += part[(int64_t)(t + 2) * R * R + pr];
      s3 += part[(int64_t)(t + 3) * R * R + pr];
    }
    for (; t < tiles; ++t) s0 += part[(int64_t)t * R * R + pr];
    G[pr] = (s0 + s1) + (s2 + s3);
  }
}

}  // namespace

size_t gram_part_doubles(int maxn, int R, int r) {
  return (size_t)r * 3 * ((maxn + kRT - 1) / kRT) * R * R;
}

cudaError_t launch_gram_tiles(const GramArgs& g, cudaStream_t st) {
  gram_tiles_kernel<<<dim3(g.tmax, 3, g.r), kRT, 0, st>>>(g);
  gram_combine_kernel<<<dim3(3, g.r), 256, 0, st>>>(g);
  return cudaGetLastError();
}

int gram_tiles_for(int n) { return (n + kRT - 1) / kRT; }

cudaError_t launch_als_rows_commit(const RowsAls& a, cudaStream_t st) {
  als_commit_stop_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pad_factors(const RowsAls& a, cudaStream_t st) {
  if (!a.Up[0]) return cudaSuccess;
  pad_factors_kernel<<<dim3(64, 3, a.r), kRT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_als_rows_mode(const RowsAls& a, int mode, cudaStream_t st) {
  const int n = mode == 0 ? a.nI : mode == 1 ? a.nJ : a.nK;
  const int ntile = (n + kRT - 1) / kRT;
  als_vinv_kernel<<<a.r, 32, 0, st>>>(a, mode);
  switch (a.R <= 4 ? 4 : a.R <= 8 ? 8 : a.R <= 12 ? 12 : a.R <= 16 ? 16 : 0) {
    case 4: als_rows_kernel<4><<<dim3(ntile, a.r), kRT, 0, st>>>(a, mode); break;
    case 8: als_rows_kernel<8><<<dim3(ntile, a.r), kRT, 0, st>>>(a, mode); break;
    case 12: als_rows_kernel<12><<<dim3(ntile, a.r), kRT, 0, st>>>(a, mode); break;
    case 16: als_rows_kernel<16><<<dim3(ntile, a.r), kRT, 0, st>>>(a, mode); break;
    default: return cudaErrorInvalidValue;
  }
  als_reduce_kernel<<<a.r, 256, 0, st>>>(a, mode);
  als_scale_kernel<<<dim3(ntile, a.r), kRT, 0, st>>>(a, mode);
  return cudaGetLastError();
}

size_t als_rows_part_doubles(int maxn, int R, int r) {
  return (size_t)r * ((maxn + kRT - 1) / kRT) * (R * R + 1);
}

}  // namespace sbt
