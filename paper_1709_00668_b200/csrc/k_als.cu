// k_als.cu -- a4: batched CP-ALS on the r dense summaries (Alg. 1 l.5 P:213; R10-R12).
//
// Per repetition rho (grid.y / block index), per iteration, for modes 0, 1, 2:
//     M = MTTKRP_m(Y; U_others)   V = *_{n != m} U_n^T U_n   U_m = M V^{-1}
//     lambda_f = ||U_m(:, f)||_2,  U_m(:, f) /= lambda_f
// MTTKRP uses the two-pass sweep: pass 1 streams Y once for M_0 (Khatri-Rao rows formed on
// the fly in shared memory); pass 2 streams Y once for D(u,q,f) = sum_p Y(u,q,p) U_0(p,f)
// (with the NEW U_0), from which M_1(q,f) = sum_u D U_2 and, after U_1 is solved,
// M_2(u,f) = sum_q D U_1_new are small contractions.  This is the same arithmetic as three
// separate MTTKRPs (U_0 is fixed between them) with 2 instead of 3 passes over Y.
// Precision: fp32 products, fp32 runs of <= 32 terms combined in fp64; Grams, the R x R
// solve (Cholesky, pseudo-inverse fallback), norms and the fit in fp64; factors stored fp32.
#include "common.cuh"
#include "internal.h"
#include "als_small.cuh"

namespace sbt {

constexpr int kAlsThreads = 256;
constexpr int kTile0 = 32;    // rows per W tile per row-slot in mttkrp0

__host__ __device__ inline int rb4(int rb) { return (rb + 3) & ~3; }

// ---------------------------------------------------------------------------------------
// init: Philox U(0,1) factors rounded to fp32 (R10) and per-rep state
// ---------------------------------------------------------------------------------------
__global__ void als_init_kernel(DenseAls a, uint64_t seed, uint32_t update_id, uint32_t rep0,
                                int init_factors, uint32_t rep_stride) {
  const int m = blockIdx.y, rep = blockIdx.z;
  const int n = m == 0 ? a.nI : m == 1 ? a.nJ : a.nK;
  const int64_t tot = (int64_t)n * a.R;
  if (init_factors) {
    float* U = a.U[m] + rep * a.u_stride[m];
    // global repetition index (a rank owning reps rank, rank + G, ... passes rep_stride = G)
    const uint32_t w3 = ctr_word3(kDomainAlsInit, rep0 + rep * rep_stride, m);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
         e += (int64_t)gridDim.x * blockDim.x) {
      const U4 o = philox4x32_10(U4{(uint32_t)e, 0u, update_id, w3}, (uint32_t)seed, (uint32_t)(seed >> 32));
      U[e] = __double2float_rn(uniform53(o.x, o.y));
    }
  }
  if (blockIdx.x == 0 && m == 0 && threadIdx.x == 0) {
    a.done[rep] = 0; a.iters[rep] = 0; a.fit[rep] = 0.0; a.fit_prev[rep] = 0.0; a.flags[rep] = 0;
  }
}

// Gram G = U^T U (fp64) of a stored fp32 factor [n][R]; one block.
__device__ void block_gram(const float* __restrict__ U, int n, int R, double* __restrict__ G) {
  for (int pr = threadIdx.x; pr < R * R; pr += blockDim.x) {
    const int f = pr / R, g = pr - f * R;
    if (g < f) continue;
    double s = 0.0;
    for (int row = 0; row < n; ++row)
      s += (double)U[(int64_t)row * R + f] * (double)U[(int64_t)row * R + g];
    G[f * R + g] = s;
    G[g * R + f] = s;
  }
}

__global__ void gram_kernel(DenseAls a) {
  const int m = blockIdx.x, rep = blockIdx.y;
  const int n = m == 0 ? a.nI : m == 1 ? a.nJ : a.nK;
  block_gram(a.U[m] + rep * a.u_stride[m], n, a.R, a.G + ((int64_t)rep * 3 + m) * a.R * a.R);
}

// sum of squares of Y per repetition: per-block partials, then an ordered reduction.
__global__ void sumsq_kernel(const float* __restrict__ Y, int64_t y_stride, int64_t rows,
                             int64_t pitch, int64_t ncols, int64_t rows_per_block, double* part) {
  __shared__ double sh[32];
  const int rep = blockIdx.y;
  const float* Yr = Y + rep * y_stride;
  const int64_t rb = (int64_t)blockIdx.x * rows_per_block, re = min(rb + rows_per_block, rows);
  double s = 0.0;
  const int64_t tot = (re - rb) * ncols;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int64_t row = rb + e / ncols, col = e % ncols;
    const double v = Yr[row * pitch + col];
    s += v * v;
  }
  s = block_sum_d(s, sh);
  if (threadIdx.x == 0) part[(int64_t)rep * gridDim.x + blockIdx.x] = s;
}

__global__ void sum_parts_kernel(const double* part, int nb, double* out) {
  const int rep = threadIdx.x;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(int64_t)rep * nb + b];
  out[rep] = s;
}

cudaError_t launch_sumsq_dense(const float* Y, int64_t y_stride, int64_t rows, int64_t pitch,
                               int64_t ncols, int r, double* out, cudaStream_t st) {
  // `out` must have room for r * (1 + nb) doubles: partials after the r results.
  int64_t nb = (int64_t)kNumSMs * 4 / (r > 0 ? r : 1);
  if (nb < 1) nb = 1;
  if (nb > rows) nb = rows > 0 ? rows : 1;
  if (nb > 256) nb = 256;
  const int64_t rpb = ceil_div(rows > 0 ? rows : 1, nb);
  nb = ceil_div(rows > 0 ? rows : 1, rpb);
  double* part = out + r;
  sumsq_kernel<<<dim3((unsigned)nb, (unsigned)r), 256, 0, st>>>(Y, y_stride, rows, pitch, ncols, rpb, part);
  sum_parts_kernel<<<1, r, 0, st>>>(part, (int)nb, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// pass 1: M_0 partials.  Block = (row block b, rep, column chunk z).  Thread (rr, p): column
// p of the chunk, rows rr, rr + RP, ...  W(row, f) = U_1(q,f) U_2(u,f) staged per tile.
// ---------------------------------------------------------------------------------------
template <int RB>
__global__ void __launch_bounds__(kAlsThreads) mttkrp0_kernel(DenseAls a, int cw, int RP) {
  const int rep = blockIdx.y;
  if (a.done[rep]) return;
  constexpr int S4 = (RB + 3) & ~3;
  __shared__ __align__(16) float Ws[kTile0 * 8 * S4];
  const int R = a.R, nJ = a.nJ;
  const int c0 = blockIdx.z * cw;
  const int ncol = min(cw, a.nI - c0);
  const int rr = threadIdx.x / cw, pl = threadIdx.x - rr * cw;
  const bool active = rr < RP && pl < ncol;
  const int p = c0 + pl;
  const int64_t nrows = (int64_t)a.nK * nJ;
  const int64_t rb = (int64_t)blockIdx.x * a.rows_per_block0;
  const int64_t re = min(rb + a.rows_per_block0, nrows);
  const float* Y = a.Y + rep * a.y_stride;
  const float* U1 = a.U[1] + rep * a.u_stride[1];
  const float* U2 = a.U[2] + rep * a.u_stride[2];
  const int tile = kTile0 * RP;
  float acc[RB];
  double acc64[RB];
#pragma unroll
  for (int f = 0; f < RB; ++f) { acc[f] = 0.f; acc64[f] = 0.0; }
  for (int64_t tb = rb; tb < re; tb += tile) {
    const int tn = (int)min((int64_t)tile, re - tb);
    for (int e = threadIdx.x; e < tn * S4; e += blockDim.x) {
      const int t = e / S4, f = e - t * S4;
      float w = 0.f;
      if (f < R) {
        const int64_t row = tb + t;
        const int u = (int)(row / nJ), q = (int)(row - (int64_t)u * nJ);
        w = U1[(int64_t)q * R + f] * U2[(int64_t)u * R + f];
      }
      Ws[e] = w;
    }
    __syncthreads();
    if (active) {
      const float* yp = Y + (tb + rr) * a.pitch + p;
#pragma unroll 4
      for (int t = rr; t < tn; t += RP, yp += RP * a.pitch) {
        const float y = *yp;
        const float4* w4 = reinterpret_cast<const float4*>(Ws + t * S4);
#pragma unroll
        for (int f4 = 0; f4 < S4 / 4; ++f4) {
          const float4 w = w4[f4];
          if (4 * f4 + 0 < RB) acc[4 * f4 + 0] = fmaf(y, w.x, acc[4 * f4 + 0]);
          if (4 * f4 + 1 < RB) acc[4 * f4 + 1] = fmaf(y, w.y, acc[4 * f4 + 1]);
          if (4 * f4 + 2 < RB) acc[4 * f4 + 2] = fmaf(y, w.z, acc[4 * f4 + 2]);
          if (4 * f4 + 3 < RB) acc[4 * f4 + 3] = fmaf(y, w.w, acc[4 * f4 + 3]);
        }
      }
#pragma unroll
      for (int f = 0; f < RB; ++f) { acc64[f] += (double)acc[f]; acc[f] = 0.f; }
    }
    __syncthreads();
  }
  // reduce the RP row slots of each column in shared memory (fixed order), then store
  __shared__ double red[kAlsThreads];
  double* part = a.part0 + (((int64_t)rep * a.nb0 + blockIdx.x) * a.nI) * R;
#pragma unroll
  for (int f = 0; f < RB; ++f) {
    if (f >= R) break;
    red[threadIdx.x] = active ? acc64[f] : 0.0;
    __syncthreads();
    if (rr == 0 && pl < ncol) {
      double s = 0.0;
      for (int k = 0; k < RP; ++k) s += red[k * cw + pl];
      part[(int64_t)p * R + f] = s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// pass 2: D(row, f) = sum_p Y(row, p) U_0(p, f).  One warp per 32 consecutive rows; the
// warp stages a 32 x 32 tile of Y (odd-stride smem, conflict-free) and the matching U_0
// rows, then lane l reduces row l.
// ---------------------------------------------------------------------------------------
template <int RB> struct DpassCfg { static constexpr int NW = RB <= 12 ? 8 : 4; };

template <int RB>
__global__ void __launch_bounds__(kAlsThreads) dpass_kernel(DenseAls a) {
  const int rep = blockIdx.y;
  if (a.done[rep]) return;
  constexpr int S4 = (RB + 3) & ~3;
  constexpr int NW = DpassCfg<RB>::NW;
  __shared__ float tile_sh[NW][32][33];
  __shared__ __align__(16) float uc_sh[NW][32 * S4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = a.R, nI = a.nI;
  const int64_t nrows = (int64_t)a.nK * a.nJ;
  const int64_t row0 = ((int64_t)blockIdx.x * NW + warp) * 32;
  if (row0 >= nrows) return;
  const float* Y = a.Y + rep * a.y_stride;
  const float* U0 = a.U[0] + rep * a.u_stride[0];
  float (*tile)[33] = tile_sh[warp];
  float* uc = uc_sh[warp];
  float acc[RB];
  double acc64[RB];
#pragma unroll
  for (int f = 0; f < RB; ++f) { acc[f] = 0.f; acc64[f] = 0.0; }
  const int nr = (int)min((int64_t)32, nrows - row0);
  for (int pc = 0; pc < nI; pc += 32) {
    const int w = min(32, nI - pc);
#pragma unroll 8
    for (int r2 = 0; r2 < 32; ++r2)
      tile[r2][lane] = (r2 < nr && lane < w) ? Y[(row0 + r2) * a.pitch + pc + lane] : 0.f;
#pragma unroll
    for (int f = 0; f < S4; ++f)
      uc[lane * S4 + f] = (lane < w && f < R) ? U0[(int64_t)(pc + lane) * R + f] : 0.f;
    __syncwarp();
    for (int pp = 0; pp < w; ++pp) {
      const float y = tile[lane][pp];
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
    float* D = a.D + (((int64_t)rep * nrows) + row0 + lane) * R;
#pragma unroll
    for (int f = 0; f < RB; ++f)
      if (f < R) D[f] = (float)acc64[f];
  }
}

// M_1(q, f) = sum_u D(u, q, f) U_2(u, f)   (fp64)
__global__ void m1_kernel(DenseAls a) {
  const int rep = blockIdx.y;
  if (a.done[rep]) return;
  const int R = a.R;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)a.nJ * R) return;
  const int f = (int)(idx % R);
  const int64_t nrows = (int64_t)a.nK * a.nJ;
  const float* D = a.D + (int64_t)rep * nrows * R;
  const float* U2 = a.U[2] + rep * a.u_stride[2];
  double s = 0.0;
  const int64_t step = (int64_t)a.nJ * R;
#pragma unroll 4
  for (int u = 0; u < a.nK; ++u) s += (double)D[u * step + idx] * (double)U2[(int64_t)u * R + f];
  a.M[rep * a.m_stride + idx] = s;
}

// M_2(u, f) = sum_q D(u, q, f) U_1(q, f); one block (32*R threads) per (u, rep).
__global__ void m2_kernel(DenseAls a) {
  const int u = blockIdx.x, rep = blockIdx.y;
  if (a.done[rep]) return;
  __shared__ double red[32 * kMaxR];
  const int R = a.R;
  const int64_t nrows = (int64_t)a.nK * a.nJ;
  const float* D = a.D + ((int64_t)rep * nrows + (int64_t)u * a.nJ) * R;
  const float* U1 = a.U[1] + rep * a.u_stride[1];
  const int tot = a.nJ * R;
  double s = 0.0;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) s += (double)D[idx] * (double)U1[idx];
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < R) {
    double t = 0.0;
    for (int k = threadIdx.x; k < (int)blockDim.x; k += R) t += red[k];
    a.M[rep * a.m_stride + (int64_t)u * R + threadIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------------------
// R x R solve, normalisation, Gram, fit.  One block per repetition.
// ---------------------------------------------------------------------------------------
template <int RB>
__global__ void __launch_bounds__(kAlsThreads) solve_kernel(DenseAls a, int mode) {
  const int rep = blockIdx.x;
  if (a.done[rep]) return;
  __shared__ double V[kMaxR * kMaxR];
  __shared__ double L[kMaxR * kMaxR];
  __shared__ double W1[kMaxR * kMaxR];
  __shared__ double W2[kMaxR * kMaxR];
  __shared__ double red[32];
  __shared__ double lam_s[kMaxR];
  __shared__ int use_pinv;
  const int R = a.R;
  const int n = mode == 0 ? a.nI : mode == 1 ? a.nJ : a.nK;
  double* G = a.G + (int64_t)rep * 3 * R * R;
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
    double v = 1.0;
    for (int o = 0; o < 3; ++o)
      if (o != mode) v *= G[o * R * R + idx];
    V[idx] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    use_pinv = cholesky_R(V, L, R) ? 0 : 1;
    if (use_pinv) { pinv_R(V, L, R, W1, W2); a.flags[rep] |= 1; }
  }
  __syncthreads();
  float* U = a.U[mode] + rep * a.u_stride[mode];
  double* Us = a.Uscr + rep * a.m_stride;
  const double* Msrc = a.M + rep * a.m_stride;
  double cs[RB];
#pragma unroll
  for (int f = 0; f < RB; ++f) cs[f] = 0.0;
  for (int row = threadIdx.x; row < n; row += blockDim.x) {
    double m[RB], x[RB];
    if (mode == 0) {
      const double* part = a.part0 + (int64_t)rep * a.nb0 * a.nI * R + (int64_t)row * R;
#pragma unroll
      for (int f = 0; f < RB; ++f) m[f] = 0.0;
      for (int b = 0; b < a.nb0; ++b) {
        const double* pb = part + (int64_t)b * a.nI * R;
#pragma unroll
        for (int f = 0; f < RB; ++f)
          if (f < R) m[f] += pb[f];
      }
    } else {
#pragma unroll
      for (int f = 0; f < RB; ++f) m[f] = f < R ? Msrc[(int64_t)row * R + f] : 0.0;
    }
    if (!use_pinv) {
      double y[RB];
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        if (i < R) {
          double s = m[i];
#pragma unroll
          for (int j = 0; j < i; ++j) s -= L[i * R + j] * y[j];
          y[i] = s / L[i * R + i];
        }
      }
#pragma unroll
      for (int i = RB - 1; i >= 0; --i) {
        if (i < R) {
          double s = y[i];
#pragma unroll
          for (int j = i + 1; j < RB; ++j)
            if (j < R) s -= L[j * R + i] * x[j];
          x[i] = s / L[i * R + i];
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        if (i < R) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < RB; ++j)
            if (j < R) s += L[i * R + j] * m[j];
          x[i] = s;
        }
      }
    }
#pragma unroll
    for (int f = 0; f < RB; ++f)
      if (f < R) { Us[(int64_t)row * R + f] = x[f]; cs[f] += x[f] * x[f]; }
  }
#pragma unroll
  for (int f = 0; f < RB; ++f) {
    if (f < R) {
      const double t = block_sum_d(cs[f], red);
      if (threadIdx.x == 0) lam_s[f] = sqrt(t);
    }
  }
  __syncthreads();
  double inner = 0.0;
  for (int row = threadIdx.x; row < n; row += blockDim.x) {
#pragma unroll
    for (int f = 0; f < RB; ++f) {
      if (f < R) {
        const double l = lam_s[f];
        const double un = l > 0.0 ? Us[(int64_t)row * R + f] / l : Us[(int64_t)row * R + f];
        const float uf = __double2float_rn(un);
        U[(int64_t)row * R + f] = uf;
        if (mode == 2) inner += l * (double)uf * Msrc[(int64_t)row * R + f];
      }
    }
  }
  if (threadIdx.x < R) a.lam[rep * R + threadIdx.x] = lam_s[threadIdx.x];
  __syncthreads();
  block_gram(U, n, R, G + mode * R * R);
  if (mode == 2) {
    inner = block_sum_d(inner, red);   // contains __syncthreads: Gram writes visible
    if (threadIdx.x == 0) {
      double mn = 0.0;
      for (int f = 0; f < R; ++f)
        for (int g = 0; g < R; ++g)
          mn += lam_s[f] * lam_s[g] * G[f * R + g] * G[R * R + f * R + g] * G[2 * R * R + f * R + g];
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
      if (stop) a.done[rep] = 1;
    }
  }
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
static void col_chunking(int nI, int* cw, int* nz, int* RP) {
  const int nchunks = (nI + kAlsThreads - 1) / kAlsThreads;
  *nz = nchunks;
  *cw = (nI + nchunks - 1) / nchunks;
  int rp = kAlsThreads / *cw;
  if (rp < 1) rp = 1;
  if (rp > 8) rp = 8;
  *RP = rp;
}

size_t dense_als_workspace(DenseAls* a) {
  int cw, nz, RP;
  col_chunking(a->nI, &cw, &nz, &RP);
  const int64_t nrows = (int64_t)a->nK * a->nJ;
  int64_t want = (int64_t)kNumSMs * 6 / ((int64_t)a->r * nz);
  if (want < 1) want = 1;
  const int64_t tile = (int64_t)kTile0 * RP;
  int64_t rpb = ceil_div(ceil_div(nrows, want), tile) * tile;
  if (rpb < tile) rpb = tile;
  a->rows_per_block0 = rpb;
  a->nb0 = (int)ceil_div(nrows, rpb);
  const int64_t maxn = (int64_t)max(a->nI, max(a->nJ, a->nK));
  a->m_stride = maxn * a->R;
  const int R = a->R, r = a->r;
  size_t b = 0;
  auto add = [&](size_t bytes) { b += (bytes + 255) & ~(size_t)255; };
  add(sizeof(double) * r * 3 * R * R);           // G
  add(sizeof(double) * r * R);                   // lam
  add(sizeof(double) * r * (1 + 256));           // ysq + partials
  add(sizeof(double) * r);                       // fit
  add(sizeof(double) * r);                       // fit_prev
  add(sizeof(int) * r);                          // iters
  add(sizeof(int) * r);                          // done
  add(sizeof(int) * r);                          // flags
  add(sizeof(double) * r * a->nb0 * a->nI * R);  // part0
  add(sizeof(float) * r * nrows * R);            // D
  add(sizeof(double) * r * a->m_stride);         // M
  add(sizeof(double) * r * a->m_stride);         // Uscr
  return b;
}

cudaError_t dense_als_bind_workspace(DenseAls* a, void* ws) {
  char* p = static_cast<char*>(ws);
  const int R = a->R, r = a->r;
  const int64_t nrows = (int64_t)a->nK * a->nJ;
  auto take = [&](size_t bytes) { char* q = p; p += (bytes + 255) & ~(size_t)255; return q; };
  a->G = (double*)take(sizeof(double) * r * 3 * R * R);
  a->lam = (double*)take(sizeof(double) * r * R);
  a->ysq = (double*)take(sizeof(double) * r * (1 + 256));
  a->fit = (double*)take(sizeof(double) * r);
  a->fit_prev = (double*)take(sizeof(double) * r);
  a->iters = (int*)take(sizeof(int) * r);
  a->done = (int*)take(sizeof(int) * r);
  a->flags = (int*)take(sizeof(int) * r);
  a->part0 = (double*)take(sizeof(double) * r * a->nb0 * a->nI * R);
  a->D = (float*)take(sizeof(float) * r * nrows * R);
  a->M = (double*)take(sizeof(double) * r * a->m_stride);
  a->Uscr = (double*)take(sizeof(double) * r * a->m_stride);
  return cudaSuccess;
}

cudaError_t launch_als_init(const DenseAls& a, uint64_t seed, uint32_t update_id, uint32_t rep0,
                            bool init_factors, cudaStream_t st) {
  const int maxn = max(a.nI, max(a.nJ, a.nK));
  int bx = (int)ceil_div((int64_t)maxn * a.R, 256);
  if (bx > 64) bx = 64;
  als_init_kernel<<<dim3(bx, 3, a.r), 256, 0, st>>>(a, seed, update_id, rep0, init_factors ? 1 : 0, 1u);
  gram_kernel<<<dim3(3, a.r), 256, 0, st>>>(a);
  return launch_sumsq_dense(a.Y, a.y_stride, (int64_t)a.nK * a.nJ, a.pitch, a.nI, a.r, a.ysq, st);
}

cudaError_t launch_als_init_factors(const DenseAls& a, uint64_t seed, uint32_t update_id,
                                    uint32_t rep0, cudaStream_t st, uint32_t rep_stride) {
  const int maxn = max(a.nI, max(a.nJ, a.nK));
  int bx = (int)ceil_div((int64_t)maxn * a.R, 256);
  if (bx > 64) bx = 64;
  als_init_kernel<<<dim3(bx, 3, a.r), 256, 0, st>>>(a, seed, update_id, rep0, 1, rep_stride);
  return cudaGetLastError();
}

cudaError_t launch_als_gram(const DenseAls& a, cudaStream_t st) {
  gram_kernel<<<dim3(3, a.r), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_als_solve(const DenseAls& a, int mode, cudaStream_t st) {
  if (a.R <= 4) solve_kernel<4><<<a.r, kAlsThreads, 0, st>>>(a, mode);
  else if (a.R <= 8) solve_kernel<8><<<a.r, kAlsThreads, 0, st>>>(a, mode);
  else if (a.R <= 10) solve_kernel<10><<<a.r, kAlsThreads, 0, st>>>(a, mode);
  else if (a.R <= 12) solve_kernel<12><<<a.r, kAlsThreads, 0, st>>>(a, mode);
  else if (a.R <= 16) solve_kernel<16><<<a.r, kAlsThreads, 0, st>>>(a, mode);
  else if (a.R <= 24) solve_kernel<24><<<a.r, kAlsThreads, 0, st>>>(a, mode);
  else solve_kernel<32><<<a.r, kAlsThreads, 0, st>>>(a, mode);
  return cudaGetLastError();
}

template <int RB>
static void als_iteration(const DenseAls& a, cudaStream_t st) {
  int cw, nz, RP;
  col_chunking(a.nI, &cw, &nz, &RP);
  const int threads0 = ((RP * cw + 31) / 32) * 32;
  mttkrp0_kernel<RB><<<dim3(a.nb0, a.r, nz), threads0, 0, st>>>(a, cw, RP);
  solve_kernel<RB><<<a.r, kAlsThreads, 0, st>>>(a, 0);
  const int64_t nrows = (int64_t)a.nK * a.nJ;
  constexpr int NW = DpassCfg<RB>::NW;
  dpass_kernel<RB><<<dim3((unsigned)ceil_div(nrows, 32 * NW), a.r), 32 * NW, 0, st>>>(a);
  m1_kernel<<<dim3((unsigned)ceil_div((int64_t)a.nJ * a.R, 256), a.r), 256, 0, st>>>(a);
  solve_kernel<RB><<<a.r, kAlsThreads, 0, st>>>(a, 1);
  m2_kernel<<<dim3(a.nK, a.r), 32 * a.R, 0, st>>>(a);
  solve_kernel<RB><<<a.r, kAlsThreads, 0, st>>>(a, 2);
}

template <int RB>
static cudaError_t run_als_rb(const DenseAls& a, cudaStream_t st) {
  for (int it = 0; it < a.maxit; ++it) als_iteration<RB>(a, st);
  return cudaGetLastError();
}

cudaError_t run_dense_als(const DenseAls& a, cudaStream_t st) {
  if (a.R <= 4) return run_als_rb<4>(a, st);
  if (a.R <= 8) return run_als_rb<8>(a, st);
  if (a.R <= 10) return run_als_rb<10>(a, st);
  if (a.R <= 12) return run_als_rb<12>(a, st);
  if (a.R <= 16) return run_als_rb<16>(a, st);
  if (a.R <= 24) return run_als_rb<24>(a, st);
  return run_als_rb<32>(a, st);
}

// ---------------------------------------------------------------------------------------
// single MTTKRP (stateless API): fp64 accumulation -> fp32 output
// ---------------------------------------------------------------------------------------
__global__ void reduce_part0_kernel(DenseAls a, float* M) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)a.nI * a.R;
  if (idx >= tot) return;
  double s = 0.0;
  for (int b = 0; b < a.nb0; ++b) s += a.part0[(int64_t)b * tot + idx];
  M[idx] = (float)s;
}
__global__ void m_to_f32_kernel(const double* Md, int64_t n, float* M) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < n) M[idx] = (float)Md[idx];
}

template <int RB>
static cudaError_t mttkrp_single_rb(const DenseAls& a, int mode, float* M, cudaStream_t st) {
  cudaMemsetAsync(a.done, 0, sizeof(int) * a.r, st);
  const int64_t nrows = (int64_t)a.nK * a.nJ;
  if (mode == 0) {
    int cw, nz, RP;
    col_chunking(a.nI, &cw, &nz, &RP);
    const int threads0 = ((RP * cw + 31) / 32) * 32;
    mttkrp0_kernel<RB><<<dim3(a.nb0, 1, nz), threads0, 0, st>>>(a, cw, RP);
    reduce_part0_kernel<<<(unsigned)ceil_div((int64_t)a.nI * a.R, 256), 256, 0, st>>>(a, M);
  } else {
    constexpr int NW = DpassCfg<RB>::NW;
    dpass_kernel<RB><<<dim3((unsigned)ceil_div(nrows, 32 * NW), 1), 32 * NW, 0, st>>>(a);
    if (mode == 1) {
      m1_kernel<<<dim3((unsigned)ceil_div((int64_t)a.nJ * a.R, 256), 1), 256, 0, st>>>(a);
      m_to_f32_kernel<<<(unsigned)ceil_div((int64_t)a.nJ * a.R, 256), 256, 0, st>>>(a.M, (int64_t)a.nJ * a.R, M);
    } else {
      m2_kernel<<<dim3(a.nK, 1), 32 * a.R, 0, st>>>(a);
      m_to_f32_kernel<<<(unsigned)ceil_div((int64_t)a.nK * a.R, 256), 256, 0, st>>>(a.M, (int64_t)a.nK * a.R, M);
    }
  }
  return cudaGetLastError();
}

cudaError_t dense_mttkrp_single(const DenseAls& a, int mode, float* M, cudaStream_t st) {
  if (a.R <= 4) return mttkrp_single_rb<4>(a, mode, M, st);
  if (a.R <= 8) return mttkrp_single_rb<8>(a, mode, M, st);
  if (a.R <= 10) return mttkrp_single_rb<10>(a, mode, M, st);
  if (a.R <= 12) return mttkrp_single_rb<12>(a, mode, M, st);
  if (a.R <= 16) return mttkrp_single_rb<16>(a, mode, M, st);
  if (a.R <= 24) return mttkrp_single_rb<24>(a, mode, M, st);
  return mttkrp_single_rb<32>(a, mode, M, st);
}

// ---------------------------------------------------------------------------------------
// Full-tensor CP-ALS over a time-sharded store: every rank streams its
// slab with the kernels above (r = 1); the mode-0 and mode-1 MTTKRPs are sums over slices, so
// their slab partials are all-reduced and every rank solves the replicated A, B; the mode-2
// MTTKRP rows belong to the rank holding the slice: they are all-gathered and scattered to
// their global rows, and every rank solves the replicated C.  Integer-free but deterministic:
// the all-reduce gives every rank the same bits, so the factors stay identical everywhere.
// ---------------------------------------------------------------------------------------
__global__ void reduce_part0_d_kernel(DenseAls a, double* M) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)a.nI * a.R;
  if (idx >= tot || a.done[0]) return;
  double s = 0.0;
  for (int b = 0; b < a.nb0; ++b) s += a.part0[(int64_t)b * tot + idx];   // block order, as solve_kernel
  M[idx] = s;
}
// rows of the replicated C held by this rank (kmap: local slice -> global slice)
__global__ void gather_rows_kernel(const float* C, const int32_t* kmap, int64_t nloc, int R, float* Cl) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nloc * R) return;
  const int64_t t = e / R;
  Cl[e] = C[(int64_t)kmap[t] * R + (e - t * R)];
}
// all-gathered mode-2 rows [world][kpad][R] -> their global rows of M (gidx: global slice or -1)
__global__ void scatter_rows_kernel(const double* in, const int32_t* gidx, int64_t n, int R, double* M,
                                    const int* done) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * R || done[0]) return;
  const int64_t t = e / R;
  const int g = gidx[t];
  if (g >= 0) M[(int64_t)g * R + (e - t * R)] = in[e];
}

template <int RB>
static cudaError_t als_sharded_rb(DenseAls loc, DenseAls glob, const int32_t* kmap, const int32_t* gidx,
                                  int kpad, double* stage, double* gathered, const AlsComm& c, cudaStream_t st) {
  const int R = glob.R;
  const int64_t nloc = loc.nK;
  // loc reads the replicated A, B and its own rows of C; its flags / done are glob's, and its
  // mode-1 MTTKRP partial lands in glob's M (all-reduced in place there)
  loc.done = glob.done; loc.flags = glob.flags; loc.M = glob.M;
  int cw, nz, RP;
  col_chunking(loc.nI, &cw, &nz, &RP);
  const int threads0 = ((RP * cw + 31) / 32) * 32;
  constexpr int NW = DpassCfg<RB>::NW;
  DenseAls loc2 = loc;   // mode-2 rows into the staging buffer
  loc2.M = stage;
  DenseAls g0 = glob;    // mode-0 solve reads M through part0 with one "block"
  g0.part0 = glob.M; g0.nb0 = 1;
  auto refresh_cloc = [&]() {
    if (nloc > 0)
      gather_rows_kernel<<<(unsigned)ceil_div(nloc * R, 256), 256, 0, st>>>(glob.U[2], kmap, nloc, R, loc.U[2]);
  };
  refresh_cloc();
  for (int it = 0; it < glob.maxit; ++it) {
    // mode 0: slab partials -> all-reduce -> replicated solve
    if (nloc > 0) {
      mttkrp0_kernel<RB><<<dim3(loc.nb0, 1, nz), threads0, 0, st>>>(loc, cw, RP);
      reduce_part0_d_kernel<<<(unsigned)ceil_div((int64_t)loc.nI * R, 256), 256, 0, st>>>(loc, glob.M);
    } else {
      cudaMemsetAsync(glob.M, 0, sizeof(double) * loc.nI * R, st);
    }
    cudaError_t e = c.sum_d(c.ctx, glob.M, (size_t)glob.nI * R, st);
    if (e != cudaSuccess) return e;
    solve_kernel<RB><<<1, kAlsThreads, 0, st>>>(g0, 0);
    // mode 1: D of the slab, M_1 partial -> all-reduce -> replicated solve
    if (nloc > 0) {
      const int64_t nrows = nloc * loc.nJ;
      dpass_kernel<RB><<<dim3((unsigned)ceil_div(nrows, 32 * NW), 1), 32 * NW, 0, st>>>(loc);
      m1_kernel<<<dim3((unsigned)ceil_div((int64_t)loc.nJ * R, 256), 1), 256, 0, st>>>(loc);
    } else {
      cudaMemsetAsync(glob.M, 0, sizeof(double) * loc.nJ * R, st);
    }
    e = c.sum_d(c.ctx, glob.M, (size_t)glob.nJ * R, st);
    if (e != cudaSuccess) return e;
    solve_kernel<RB><<<1, kAlsThreads, 0, st>>>(glob, 1);
    // mode 2: the slab's rows -> all-gather -> global rows -> replicated solve
    cudaMemsetAsync(stage, 0, sizeof(double) * (size_t)kpad * R, st);
    if (nloc > 0) m2_kernel<<<dim3((unsigned)nloc, 1), 32 * R, 0, st>>>(loc2);
    e = c.gather_d(c.ctx, stage, gathered, (size_t)kpad * R, st);
    if (e != cudaSuccess) return e;
    const int64_t ng = (int64_t)c.world * kpad;
    scatter_rows_kernel<<<(unsigned)ceil_div(ng * R, 256), 256, 0, st>>>(gathered, gidx, ng, R, glob.M, glob.done);
    solve_kernel<RB><<<1, kAlsThreads, 0, st>>>(glob, 2);
    refresh_cloc();
  }
  return cudaGetLastError();
}

cudaError_t run_dense_als_sharded(const DenseAls& loc, const DenseAls& glob, const int32_t* kmap,
                                  const int32_t* gidx, int kpad, double* stage, double* gathered,
                                  const AlsComm& c, cudaStream_t st) {
  if (glob.R <= 4) return als_sharded_rb<4>(loc, glob, kmap, gidx, kpad, stage, gathered, c, st);
  if (glob.R <= 8) return als_sharded_rb<8>(loc, glob, kmap, gidx, kpad, stage, gathered, c, st);
  if (glob.R <= 10) return als_sharded_rb<10>(loc, glob, kmap, gidx, kpad, stage, gathered, c, st);
  if (glob.R <= 12) return als_sharded_rb<12>(loc, glob, kmap, gidx, kpad, stage, gathered, c, st);
  if (glob.R <= 16) return als_sharded_rb<16>(loc, glob, kmap, gidx, kpad, stage, gathered, c, st);
  if (glob.R <= 24) return als_sharded_rb<24>(loc, glob, kmap, gidx, kpad, stage, gathered, c, st);
  return als_sharded_rb<32>(loc, glob, kmap, gidx, kpad, stage, gathered, c, st);
}

// the replicated factors' small state (no D / part0): G, lam, ysq, fit, fit_prev, iters, done,
// flags, M and Uscr sized for max(nI, nJ, nK) rows
size_t dense_als_small_workspace(const DenseAls& a) {
  const int64_t maxn = (int64_t)max(a.nI, max(a.nJ, a.nK));
  const int R = a.R;
  size_t b = 0;
  auto add = [&](size_t bytes) { b += (bytes + 255) & ~(size_t)255; };
  add(sizeof(double) * 3 * R * R); add(sizeof(double) * R); add(sizeof(double) * (1 + 256));
  add(sizeof(double)); add(sizeof(double)); add(sizeof(int)); add(sizeof(int)); add(sizeof(int));
  add(sizeof(double) * maxn * R); add(sizeof(double) * maxn * R);
  return b;
}

void dense_als_small_bind(DenseAls* a, void* ws) {
  char* p = static_cast<char*>(ws);
  const int R = a->R;
  const int64_t maxn = (int64_t)max(a->nI, max(a->nJ, a->nK));
  auto take = [&](size_t bytes) { char* q = p; p += (bytes + 255) & ~(size_t)255; return q; };
  a->G = (double*)take(sizeof(double) * 3 * R * R);
  a->lam = (double*)take(sizeof(double) * R);
  a->ysq = (double*)take(sizeof(double) * (1 + 256));
  a->fit = (double*)take(sizeof(double));
  a->fit_prev = (double*)take(sizeof(double));
  a->iters = (int*)take(sizeof(int));
  a->done = (int*)take(sizeof(int));
  a->flags = (int*)take(sizeof(int));
  a->m_stride = maxn * R;
  a->M = (double*)take(sizeof(double) * maxn * R);
  a->Uscr = (double*)take(sizeof(double) * maxn * R);
  a->part0 = nullptr; a->nb0 = 0; a->D = nullptr;
}

}  // namespace sbt
