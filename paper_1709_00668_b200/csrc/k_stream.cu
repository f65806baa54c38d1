// k_stream.cu -- full-tensor streaming passes over the dense store, HBM-bound:
//   a1  marginals (measure of importance, Eq. 1; R1, R7): fixed-point int64 sums
//       x1[i], x2[j], x3[k] of q(x) = RNE(phi(x) 2^S);
//   a7  fit: <X, [[lam; A, B, C]]> and ||X||^2 in one pass.
//
// Data path: persistent CTAs (one per SM and column chunk), each owning a contiguous range of
// rows (j,k) of the store X[k][j][0..pitch), stream their rows through a ring of ns shared-
// memory stages filled by the bulk-copy engine (cp.async.bulk + mbarrier, one producer
// thread), so each SM keeps ~100-190 KB of loads in flight with no register cost (a plain
// ring read of this kind measured 5.7 TB/s on the B200, tools/micro/bw.cu).
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace sbt {

namespace {

constexpr int kST = 512;          // threads per CTA
constexpr int kNW = kST / 32;

__device__ __forceinline__ unsigned s_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void s_mbar_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void s_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void s_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "SW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra SW_%=;\n}\n" ::"r"(s_u32(b)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void s_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(b))
      : "memory");
}
__device__ __forceinline__ void s_fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Row-range / column-chunk geometry shared by host and device.
struct StreamGeom {
  int64_t row0, nrows;      // rows (k*J + j) of the pass
  int64_t rows_per_cta;
  int pitch;                // floats per row in the store (multiple of 4)
  int cw;                   // column chunk width (floats, multiple of 4)
  int ncol;                 // real columns (I)
  int tr;                   // rows per stage
  int ns;                   // stages in the ring (<= kMaxNS)
};

constexpr int kMaxNS = 8;

// stage s of this CTA covers rows [rb + s*tr, ...); issued by one thread
__device__ __forceinline__ void ring_issue(float* ring, unsigned long long* bars, const StreamGeom& g,
                                           const float* X, int64_t rb, int64_t re, int c0, int s) {
  const int64_t r0 = rb + (int64_t)s * g.tr;
  const int nr = (int)min((int64_t)g.tr, re - r0);
  const int slot = s % g.ns;
  float* dst = ring + (size_t)slot * g.tr * g.cw;
  const int w = min(g.cw, g.pitch - c0);   // floats copied per row (multiple of 4)
  const unsigned row_bytes = (unsigned)(w * sizeof(float));
  s_expect(&bars[slot], row_bytes * nr);
  if (g.cw == g.pitch) {
    s_bulk(dst, X + r0 * g.pitch, row_bytes * nr, &bars[slot]);
  } else {
    for (int r = 0; r < nr; ++r)
      s_bulk(dst + (size_t)r * g.cw, X + (r0 + r) * g.pitch + c0, row_bytes, &bars[slot]);
  }
}

template <int MOI>
__device__ __forceinline__ long long quant(float x, float scf, double scd) {
  if (MOI == 0) {
    return __float2ll_rn(fabsf(x) * scf);      // exact product (power-of-two scale)
  } else {
    const double d = (double)x;
    return __double2ll_rn(__dmul_rn(__dmul_rn(d, d), scd));   // d*d exact (48 bits)
  }
}

// ---------------------------------------------------------------------------------------
// a1: marginals.  A warp handles kRPW consecutive rows of a stage at a time: lane l takes the
// quads l, l+32, ... (<= kMQ) of the column chunk (<= 512 floats) and keeps their x1 column
// sums in registers (int64); the kRPW row totals are reduced by one interleaved butterfly
// (kRPW independent shuffle chains) -> x2[j] (global atomic) and a CTA-local x3 window
// flushed at the end; x1 is combined across warps in shared memory (one global atomic per
// column).  Integer sums: exact and independent of the order.
// ---------------------------------------------------------------------------------------
constexpr int kX3Win = 64;
constexpr int kMQ = 4;            // quads per lane: column chunk <= 32 * 4 * 4 = 512 floats
constexpr int kRPW = 2;           // rows per warp per step
constexpr int kMargCTAs = 1;      // CTAs per SM

template <int MOI>
__global__ void __launch_bounds__(kST, kMargCTAs) marg_stream_kernel(const float* __restrict__ X, StreamGeom g,
                                                             int J, float scf, double scd,
                                                             unsigned long long* __restrict__ x1,
                                                             unsigned long long* __restrict__ x2,
                                                             unsigned long long* __restrict__ x3) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned long long bars[kMaxNS];
  __shared__ unsigned long long x3w[kX3Win];
  __shared__ unsigned long long x1s[4 * 32 * kMQ];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c0 = blockIdx.y * g.cw;
  const int cw_real = min(g.cw, g.ncol - c0);
  const int64_t rb = g.row0 + (int64_t)blockIdx.x * g.rows_per_cta;
  const int64_t re = min(rb + g.rows_per_cta, g.row0 + g.nrows);
  if (rb >= re) return;
  float* ring = reinterpret_cast<float*>(smem);
  const int nst = (int)((re - rb + g.tr - 1) / g.tr);
  const int64_t kfirst = rb / J;
  const bool x3_local = ((re - 1) / J - kfirst) < kX3Win;
  if (tid == 0) {
    for (int s = 0; s < g.ns; ++s) s_mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int s = tid; s < kX3Win; s += kST) x3w[s] = 0;
  for (int s = tid; s < 4 * 32 * kMQ; s += kST) x1s[s] = 0;
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < nst && s < g.ns; ++s) ring_issue(ring, bars, g, X, rb, re, c0, s);
  long long acc[kMQ][4];
#pragma unroll
  for (int m = 0; m < kMQ; ++m)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[m][e] = 0;
  for (int s = 0; s < nst; ++s) {
    const int64_t r0 = rb + (int64_t)s * g.tr;
    const int nr = (int)min((int64_t)g.tr, re - r0);
    const int slot = s % g.ns;
    s_wait(&bars[slot], (unsigned)(s / g.ns) & 1u);
    const float* st = ring + (size_t)slot * g.tr * g.cw;
    for (int rw = warp * kRPW; rw < nr; rw += kNW * kRPW) {
      long long rs[kRPW];
#pragma unroll
      for (int v = 0; v < kRPW; ++v) {
        rs[v] = 0;
        const int r = rw + v;
        if (r < nr) {
          const float* rowp = st + (size_t)r * g.cw;
#pragma unroll
          for (int m = 0; m < kMQ; ++m) {
            const int col = 4 * (lane + 32 * m);
            if (col < cw_real) {
              const float4 x = *reinterpret_cast<const float4*>(rowp + col);
              long long q0 = quant<MOI>(x.x, scf, scd), q1 = quant<MOI>(x.y, scf, scd);
              long long q2 = quant<MOI>(x.z, scf, scd), q3 = quant<MOI>(x.w, scf, scd);
              if (col + 1 >= cw_real) q1 = 0;
              if (col + 2 >= cw_real) q2 = 0;
              if (col + 3 >= cw_real) q3 = 0;
              acc[m][0] += q0; acc[m][1] += q1; acc[m][2] += q2; acc[m][3] += q3;
              rs[v] += (q0 + q1) + (q2 + q3);
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int v = 0; v < kRPW; ++v) rs[v] += __shfl_xor_sync(0xffffffffu, rs[v], o);
      if (lane < kRPW) {
        long long mine = rs[0];
#pragma unroll
        for (int v = 1; v < kRPW; ++v)
          if (lane == v) mine = rs[v];
        const int r = rw + lane;
        if (r < nr && mine) {
          const int64_t row = r0 + r;
          const int64_t k = row / J, j = row - k * J;
          atomicAdd(&x2[j], (unsigned long long)mine);
          if (x3_local) atomicAdd(&x3w[k - kfirst], (unsigned long long)mine);
          else atomicAdd(&x3[k], (unsigned long long)mine);
        }
      }
    }
    __syncthreads();   // stage consumed by every warp
    if (tid == 0 && s + g.ns < nst) {
      s_fence_async();
      ring_issue(ring, bars, g, X, rb, re, c0, s + g.ns);
    }
  }
#pragma unroll
  for (int m = 0; m < kMQ; ++m)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int col = 4 * (lane + 32 * m) + e;
      if (col < cw_real && acc[m][e]) atomicAdd(&x1s[col], (unsigned long long)acc[m][e]);
    }
  __syncthreads();
  for (int c = tid; c < cw_real; c += kST)
    if (x1s[c]) atomicAdd(&x1[c0 + c], x1s[c]);
  if (x3_local)
    for (int s = tid; s < kX3Win; s += kST)
      if (x3w[s]) atomicAdd(&x3[kfirst + s], x3w[s]);
}

// ---------------------------------------------------------------------------------------
// a7: fit.  inner = sum_{i,j,k} X(i,j,k) m(i,j,k), m = sum_f lam_f A(i,f) B(j,f) C(k,f);
// sq = sum X^2.  Thread t owns the column quad t % NQ of the rows of its row group t / NQ
// and holds lam_f A(i,f) for its 4 columns in registers; W(row,f) = B(j,f) C(k,f) of stage
// s+1 is formed in a double-buffered shared array while stage s is consumed (one barrier per
// stage).  fp32 per element and per stage, fp64 across stages; per-CTA partials reduced in a
// fixed order by fit_combine_kernel.
// ---------------------------------------------------------------------------------------
template <int RB>
__global__ void __launch_bounds__(kST, 1) fit_stream_kernel(const float* __restrict__ X, StreamGeom g,
                                                            int J, int R, const float* __restrict__ lam,
                                                            const float* __restrict__ A,
                                                            const float* __restrict__ B,
                                                            const float* __restrict__ C,
                                                            double* __restrict__ part,
                                                            const int32_t* __restrict__ kmap) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned long long bars[kMaxNS];
  __shared__ double red[32];
  const int tid = threadIdx.x;
  const int c0 = blockIdx.y * g.cw;
  const int cw_real = min(g.cw, g.ncol - c0);
  const int NQ = g.cw / 4;
  const int NG = kST / NQ > 0 ? kST / NQ : 1;
  const int quad = tid % NQ, grp = tid / NQ;
  const bool active = grp < NG && tid < NQ * NG;
  const int64_t rb = g.row0 + (int64_t)blockIdx.x * g.rows_per_cta;
  const int64_t re = min(rb + g.rows_per_cta, g.row0 + g.nrows);
  float* ring = reinterpret_cast<float*>(smem);
  float* Wbuf = ring + (size_t)g.ns * g.tr * g.cw;   // [2][tr][RB]
  const int nst = rb < re ? (int)((re - rb + g.tr - 1) / g.tr) : 0;
  auto build_w = [&](int s) {   // W rows of stage s: 32-bit (j,k) walk, no divisions per element
    float* W = Wbuf + (size_t)(s & 1) * g.tr * RB;
    const int64_t r0 = rb + (int64_t)s * g.tr;
    const int nr = (int)min((int64_t)g.tr, re - r0);
    const int k0 = (int)(r0 / J), j0 = (int)(r0 - (int64_t)k0 * J);
    for (int e = tid; e < nr * RB; e += kST) {
      const int r = e / RB, f = e - r * RB;
      int j = j0 + r, k = k0;
      while (j >= J) { j -= J; ++k; }
      const int64_t kg = kmap ? kmap[k] : k;
      W[e] = f < R ? B[(int64_t)j * R + f] * C[kg * R + f] : 0.f;
    }
  };
  if (tid == 0) {
    for (int s = 0; s < g.ns; ++s) s_mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (nst > 0) build_w(0);
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < nst && s < g.ns; ++s) ring_issue(ring, bars, g, X, rb, re, c0, s);
  const int col = 4 * quad;
  float al[4][RB];
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int f = 0; f < RB; ++f) {
      const int i = c0 + col + e;
      al[e][f] = (active && col + e < cw_real && f < R) ? lam[f] * A[(int64_t)i * R + f] : 0.f;
    }
  double inner = 0.0, sq = 0.0;
  for (int s = 0; s < nst; ++s) {
    const int64_t r0 = rb + (int64_t)s * g.tr;
    const int nr = (int)min((int64_t)g.tr, re - r0);
    const int slot = s % g.ns;
    if (s + 1 < nst) build_w(s + 1);   // the other W buffer (free since the last barrier)
    s_wait(&bars[slot], (unsigned)(s / g.ns) & 1u);
    if (active && col < cw_real) {
      const float* st = ring + (size_t)slot * g.tr * g.cw + col;
      const float* W = Wbuf + (size_t)(s & 1) * g.tr * RB;
      float fi = 0.f, fs = 0.f;
#pragma unroll 2
      for (int r = grp; r < nr; r += NG) {
        const float4 v = *reinterpret_cast<const float4*>(st + (size_t)r * g.cw);
        const float* w = W + r * RB;
        float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
#pragma unroll
        for (int f4 = 0; f4 < RB / 4; ++f4) {
          const float4 wv = *reinterpret_cast<const float4*>(w + 4 * f4);
          const float ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int f = 4 * f4 + t;
            m0 = fmaf(al[0][f], ww[t], m0);
            m1 = fmaf(al[1][f], ww[t], m1);
            m2 = fmaf(al[2][f], ww[t], m2);
            m3 = fmaf(al[3][f], ww[t], m3);
          }
        }
        fi = fmaf(v.x, m0, fmaf(v.y, m1, fmaf(v.z, m2, fmaf(v.w, m3, fi))));
        // padding columns are zero in the store (and carry al == 0)
        fs = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, fs))));
      }
      inner += (double)fi;
      sq += (double)fs;
    }
    __syncthreads();   // stage and W(s) consumed, W(s+1) complete
    if (tid == 0 && s + g.ns < nst) {
      s_fence_async();
      ring_issue(ring, bars, g, X, rb, re, c0, s + g.ns);
    }
  }
  inner = block_sum_d(inner, red);
  sq = block_sum_d(sq, red);
  if (tid == 0) {
    const int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    part[2 * b] = inner;
    part[2 * b + 1] = sq;
  }
}

// Grams of the three factors (fp64, fixed order): block m stages rows of factor m in shared
// memory; thread (pair, segment) accumulates, segments summed in order.
__global__ void gram3_kernel(const float* A, const float* B, const float* C, int64_t I, int64_t J,
                             int64_t K, int R, double* G /* [3][R][R] */) {
  __shared__ float rows[1024 * 8];
  __shared__ double segsum[512];
  const int m = blockIdx.x;
  const float* U = m == 0 ? A : m == 1 ? B : C;
  const int64_t n = m == 0 ? I : m == 1 ? J : K;
  const int npair = R * (R + 1) / 2;
  const int nseg = blockDim.x / npair > 0 ? blockDim.x / npair : 1;
  const int pair = threadIdx.x % npair, seg = threadIdx.x / npair;
  int f = 0, gg = pair;
  while (gg >= R - f) { gg -= R - f; ++f; }
  gg += f;
  const int64_t chunk_rows = (int64_t)(sizeof(rows) / sizeof(float)) / R;
  double acc = 0.0;
  for (int64_t c0 = 0; c0 < n; c0 += chunk_rows) {
    const int64_t nr = min(chunk_rows, n - c0);
    __syncthreads();
    for (int64_t e = threadIdx.x; e < nr * R; e += blockDim.x) rows[e] = U[c0 * R + e];
    __syncthreads();
    if (seg < nseg && threadIdx.x < nseg * npair) {
      const int64_t per = (nr + nseg - 1) / nseg;
      const int64_t a = seg * per, b = min(nr, a + per);
      for (int64_t r = a; r < b; ++r) acc += (double)rows[r * R + f] * (double)rows[r * R + gg];
    }
  }
  __syncthreads();
  if (threadIdx.x < nseg * npair) segsum[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < npair) {
    double s = 0.0;
    for (int k = 0; k < nseg; ++k) s += segsum[k * npair + threadIdx.x];
    G[(int64_t)m * R * R + f * R + gg] = s;
    G[(int64_t)m * R * R + gg * R + f] = s;
  }
}

__global__ void fit_combine_kernel(const double* part, int nb, const double* G, const float* lam,
                                   int R, double* relerr) {
  if (threadIdx.x != 0) return;
  double inner = 0.0, sq = 0.0, mn = 0.0;
  for (int b = 0; b < nb; ++b) { inner += part[2 * b]; sq += part[2 * b + 1]; }
  for (int f = 0; f < R; ++f)
    for (int g = 0; g < R; ++g)
      mn += (double)lam[f] * (double)lam[g] * G[f * R + g] * G[R * R + f * R + g] * G[2 * R * R + f * R + g];
  const double res = fmax(0.0, sq - 2.0 * inner + mn);
  *relerr = sq > 0.0 ? sqrt(res / sq) : 0.0;
}

// Geometry: column chunks of <= max_cw floats; stages of ~stage_bytes (whole rows), a ring of
// ring_bytes / stage; one CTA per SM and chunk over contiguous row ranges.
StreamGeom make_geom(const DenseView& X, int64_t row0, int64_t nrows, int* grid_x, int* grid_y,
                     int max_cw, int stage_bytes, int ring_bytes, int min_tr, int ctas_per_sm = 1) {
  StreamGeom g{};
  g.row0 = row0;
  g.nrows = nrows;
  g.pitch = (int)X.pitch;
  g.ncol = (int)X.I;
  if (g.pitch <= max_cw) {
    g.cw = g.pitch;
  } else {   // equal chunks, multiples of 4 floats
    const int nch = (g.pitch + max_cw - 1) / max_cw;
    g.cw = ((g.pitch + nch - 1) / nch + 3) & ~3;
  }
  const int nchunk = (g.pitch + g.cw - 1) / g.cw;
  g.tr = stage_bytes / (int)(g.cw * sizeof(float));
  if (g.tr < min_tr) g.tr = min_tr;
  if (g.tr > 256) g.tr = 256;
  g.ns = ring_bytes / (int)(g.tr * g.cw * sizeof(float));
  if (g.ns > kMaxNS) g.ns = kMaxNS;
  if (g.ns < 2) g.ns = 2;
  int64_t nx = (int64_t)kNumSMs * ctas_per_sm / nchunk;
  if (nx < 1) nx = 1;
  if (nx > ceil_div(nrows, 2 * g.tr)) nx = ceil_div(nrows, 2 * g.tr);   // a few stages per CTA
  if (nx < 1) nx = 1;
  g.rows_per_cta = ceil_div(nrows, nx);
  *grid_x = (int)ceil_div(nrows, g.rows_per_cta);
  *grid_y = nchunk;
  return g;
}

size_t ring_smem(const StreamGeom& g) { return sizeof(float) * (size_t)g.ns * g.tr * g.cw; }

constexpr int kRingBytes = 192 * 1024;

StreamGeom marg_geom(const DenseView& X, int64_t k0, int64_t nk, int* gx, int* gy) {
  // rows per stage: a multiple of kRPW * warps keeps every warp busy
  return make_geom(X, k0 * X.J, nk * X.J, gx, gy, 4 * 32 * kMQ, 64 * 1024, kRingBytes, kRPW * kNW,
                   kMargCTAs);
}
StreamGeom fit_geom(const DenseView& X, int* gx, int* gy) {
  return make_geom(X, 0, X.J * X.K, gx, gy, 2048, 32 * 1024, 176 * 1024, 1);
}

}  // namespace

size_t gram3_ws_doubles(int64_t I, int64_t J, int64_t K, int R) {
  return gram_part_doubles((int)std::max(I, std::max(J, K)), R, 1);
}

// Grams of three factors (fp64 [3][R][R]) with tile partials in ws (gram3_ws_doubles).
cudaError_t launch_gram3(const float* A, const float* B, const float* C, int64_t I, int64_t J,
                         int64_t K, int R, double* G, double* ws, cudaStream_t st) {
  GramArgs g{};
  g.U[0] = A; g.U[1] = B; g.U[2] = C;
  g.n[0] = (int)I; g.n[1] = (int)J; g.n[2] = (int)K;
  g.R = R; g.r = 1;
  g.tmax = gram_tiles_for((int)std::max(I, std::max(J, K)));
  g.part = ws; g.G = G; g.g_stride = 3 * R * R;
  return launch_gram_tiles(g, st);
}

bool stream_supported(const DenseView& X) {
  return X.pitch % 4 == 0 && ((uintptr_t)X.base & 15) == 0 && X.I >= 1 && X.I <= 8192 && X.J >= 1;
}

cudaError_t launch_marginals_stream(const DenseView& X, int64_t k0, int64_t nk, int moi, int S,
                                    int64_t* x1, int64_t* x2, int64_t* x3, cudaStream_t st) {
  if (nk <= 0) return cudaSuccess;
  int gx, gy;
  StreamGeom g = marg_geom(X, k0, nk, &gx, &gy);
  const float scf = ldexpf(1.0f, S < -126 ? -126 : (S > 127 ? 127 : S));
  const double scd = ldexp(1.0, S);
  const size_t smem = ring_smem(g);
  auto* u1 = reinterpret_cast<unsigned long long*>(x1);
  auto* u2 = reinterpret_cast<unsigned long long*>(x2);
  auto* u3 = reinterpret_cast<unsigned long long*>(x3);
  if (moi == 0) {
    cudaFuncSetAttribute(marg_stream_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    marg_stream_kernel<0><<<dim3(gx, gy), kST, smem, st>>>(X.base, g, (int)X.J, scf, scd, u1, u2, u3);
  } else {
    cudaFuncSetAttribute(marg_stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    marg_stream_kernel<1><<<dim3(gx, gy), kST, smem, st>>>(X.base, g, (int)X.J, scf, scd, u1, u2, u3);
  }
  return cudaGetLastError();
}

size_t fit_stream_ws_doubles(const DenseView& X) {
  int gx, gy;
  fit_geom(X, &gx, &gy);
  return 2 * (size_t)gx * gy + 3 * kMaxR * kMaxR + 8 + gram3_ws_doubles(X.I, X.J, X.K, kMaxR);
}

template <int RB>
static cudaError_t fit_stream_rb(const DenseView& X, const float* lam, const float* A, const float* B,
                                 const float* C, int R, double* ws, double* relerr, cudaStream_t st) {
  int gx, gy;
  StreamGeom g = fit_geom(X, &gx, &gy);
  const size_t smem = ring_smem(g) + sizeof(float) * 2 * (size_t)g.tr * RB;
  cudaFuncSetAttribute(fit_stream_kernel<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double* part = ws;
  double* G = ws + 2 * (size_t)gx * gy;
  fit_stream_kernel<RB><<<dim3(gx, gy), kST, smem, st>>>(X.base, g, (int)X.J, R, lam, A, B, C, part,
                                                          nullptr);
  cudaError_t e = launch_gram3(A, B, C, X.I, X.J, X.K, R, G, G + 3 * kMaxR * kMaxR, st);
  if (e != cudaSuccess) return e;
  fit_combine_kernel<<<1, 32, 0, st>>>(part, gx * gy, G, lam, R, relerr);
  return cudaGetLastError();
}

__global__ void sum_pairs_kernel(const double* part, int nb, double* out2) {
  if (threadIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int i = 0; i < nb; ++i) { a += part[2 * i]; b += part[2 * i + 1]; }
  out2[0] = a;
  out2[1] = b;
}

__global__ void fit_finish_kernel(const double* in2, const double* G, const float* lam, int R,
                                  double* relerr) {
  if (threadIdx.x != 0) return;
  double mn = 0.0;
  for (int f = 0; f < R; ++f)
    for (int g = 0; g < R; ++g)
      mn += (double)lam[f] * (double)lam[g] * G[f * R + g] * G[R * R + f * R + g] * G[2 * R * R + f * R + g];
  const double sq = in2[1];
  const double res = fmax(0.0, sq - 2.0 * in2[0] + mn);
  *relerr = sq > 0.0 ? sqrt(res / sq) : 0.0;
}

template <int RB>
static cudaError_t fit_partial_rb(const DenseView& X, const float* lam, const float* A, const float* B,
                                  const float* C, int R, const int32_t* kmap, double* ws, double* out2,
                                  cudaStream_t st) {
  int gx, gy;
  StreamGeom g = fit_geom(X, &gx, &gy);
  const size_t smem = ring_smem(g) + sizeof(float) * 2 * (size_t)g.tr * RB;
  cudaFuncSetAttribute(fit_stream_kernel<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fit_stream_kernel<RB><<<dim3(gx, gy), kST, smem, st>>>(X.base, g, (int)X.J, R, lam, A, B, C, ws, kmap);
  sum_pairs_kernel<<<1, 32, 0, st>>>(ws, gx * gy, out2);
  return cudaGetLastError();
}

cudaError_t launch_fit_stream_partial(const DenseView& X, const float* lam, const float* A, const float* B,
                                      const float* C, int R, const int32_t* kmap, double* ws,
                                      double* out2, cudaStream_t st) {
  if (X.K <= 0) {   // nothing stored here
    return cudaMemsetAsync(out2, 0, 2 * sizeof(double), st);
  }
  if (R <= 4) return fit_partial_rb<4>(X, lam, A, B, C, R, kmap, ws, out2, st);
  if (R <= 8) return fit_partial_rb<8>(X, lam, A, B, C, R, kmap, ws, out2, st);
  if (R <= 12) return fit_partial_rb<12>(X, lam, A, B, C, R, kmap, ws, out2, st);
  if (R <= 16) return fit_partial_rb<16>(X, lam, A, B, C, R, kmap, ws, out2, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_fit_finish(const double* in2, const float* lam, const float* A, const float* B,
                              const float* C, int64_t I, int64_t J, int64_t K, int R, double* ws,
                              double* relerr, cudaStream_t st) {
  cudaError_t e = launch_gram3(A, B, C, I, J, K, R, ws, ws + 3 * kMaxR * kMaxR, st);
  if (e != cudaSuccess) return e;
  fit_finish_kernel<<<1, 32, 0, st>>>(in2, ws, lam, R, relerr);
  return cudaGetLastError();
}

cudaError_t launch_fit_stream(const DenseView& X, const float* lam, const float* A, const float* B,
                              const float* C, int R, double* ws, double* relerr, cudaStream_t st) {
  if (R <= 4) return fit_stream_rb<4>(X, lam, A, B, C, R, ws, relerr, st);
  if (R <= 8) return fit_stream_rb<8>(X, lam, A, B, C, R, ws, relerr, st);
  if (R <= 12) return fit_stream_rb<12>(X, lam, A, B, C, R, ws, relerr, st);
  if (R <= 16) return fit_stream_rb<16>(X, lam, A, B, C, R, ws, relerr, st);
  return cudaErrorInvalidValue;   // callers use the tiled kernel for R > 16
}

}  // namespace sbt
