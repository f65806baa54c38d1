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
#include <stdlib.h>
#include <type_traits>

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
  int nch = 1, wpc = 1;     // marginals: column chunks per row and warps per chunk in a CTA
  int pc = 0;               // marginals: producer-consumer stage release (a producer warp)
  int dbg = 0;              // marginals: timing experiment (SBT_MARG_DBG; 1 no quantisation, 2 no work)
  int spill = 0;            // marginals Q32: warp steps between folds of the 32-bit column sums
  double qmax = 1e300;      // marginals: bound on q of the data in the pass (host part) ...
  const unsigned long long* dphi = nullptr;   // ... and a device max phi (fp64 bits) folded in
  int qpt = 1, tpg = 1, ng = 1;   // fit: quads per thread, threads per row group, row groups
  bool bres = false;              // fit: B resident in shared memory (J x kMaxR floats)
};

constexpr int kMaxNS = 8;
constexpr int kWPT = 2;           // fit: W elements per thread per stage

// marginal stages: whole rows, one bulk copy (rows are contiguous in the store)
__device__ __forceinline__ void marg_issue(float* ring, unsigned long long* bars, const StreamGeom& g,
                                           const float* X, int64_t rb, int64_t re, int s) {
  const int64_t r0 = rb + (int64_t)s * g.tr;
  const int nr = (int)min((int64_t)g.tr, re - r0);
  const int slot = s % g.ns;
  const unsigned bytes = (unsigned)((size_t)nr * g.pitch * sizeof(float));
  s_expect(&bars[slot], bytes);
  s_bulk(ring + (size_t)slot * g.tr * g.pitch, X + r0 * g.pitch, bytes, &bars[slot]);
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

template <int MOI>
__device__ __forceinline__ unsigned quant32(float x, float scf, double scd) {
  if (MOI == 0) return (unsigned)__float2uint_rn(fabsf(x) * scf);   // exact product; q < 2^31 (Q32 plan)
  const double d = (double)x;
  return (unsigned)__double2ull_rn(__dmul_rn(__dmul_rn(d, d), scd));
}

// Exact warp sum of values < 2^31 (two 16-bit halves through REDUX; each half-sum < 2^21).
__device__ __forceinline__ unsigned long long warp_sum_u31(unsigned v) {
  const unsigned lo = __reduce_add_sync(0xffffffffu, v & 0xFFFFu);
  const unsigned hi = __reduce_add_sync(0xffffffffu, v >> 16);
  return ((unsigned long long)hi << 16) + lo;
}

// ---------------------------------------------------------------------------------------
// a1: marginals.  A warp handles kRPW consecutive rows of a stage at a time: lane l takes the
// quads l, l+32, ... (<= kMQ) of the column chunk (<= 512 floats) and keeps their x1 column
// sums in registers (int64); the kRPW row totals are reduced by one interleaved butterfly
// (kRPW independent shuffle chains) -> x2[j] (global atomic) and a CTA-local x3 window
// flushed at the end; x1 is combined across warps in shared memory (one global atomic per
// column).  Integer sums: exact and independent of the order.
// ---------------------------------------------------------------------------------------
constexpr int kMQ = 4;            // quads per lane: column chunk <= 32 * 4 * 4 = 512 floats
constexpr int kRPW = 2;           // rows per warp per step
constexpr int kMargCTAs = 1;      // CTAs per SM

// Q32 (the plan bound qb <= 27: every q <= 2^27): q as uint32 (F2I.U32), a lane's 16 values of
// a row summed in 32 bits (<= 2^31), row totals by two 18-bit REDUX chunk sums, column sums in
// 32-bit registers folded into the int64 sums every g.spill warp steps (2 g.spill 2^qb < 2^32):
// about half the integer instructions per element of the 64-bit path, same exact sums.
template <int MOI, bool Q32, bool QT = true>
__global__ void __launch_bounds__(kST, kMargCTAs) marg_stream_kernel(const float* __restrict__ X, StreamGeom g,
                                                             int J, float scf, double scd,
                                                             unsigned long long* __restrict__ x1,
                                                             unsigned long long* __restrict__ x2,
                                                             unsigned long long* __restrict__ x3) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned long long bars[kMaxNS];
  __shared__ unsigned long long empty[kMaxNS];   // producer-consumer mode: stage released
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int ncons = g.nch * g.wpc;                // consumer warps
  // producer-consumer mode (g.pc): a dedicated producer warp refills a stage as soon as every
  // consumer warp has released it (an "empty" mbarrier per stage) -- no CTA-wide barrier per
  // stage, so a warp that finishes a stage early moves on to the next loaded one
  const bool producer = g.pc && warp == ncons;
  // stages hold whole rows; warp w works on column chunk w % nch of the rows w / nch,
  // w / nch + wpc, ... (kRPW at a time)
  const int chunk = warp % g.nch, wslot = warp / g.nch;
  const int c0 = chunk * g.cw;
  const int cw_real = min(g.cw, g.ncol - c0);
  const int64_t rb = g.row0 + (int64_t)blockIdx.x * g.rows_per_cta;
  const int64_t re = min(rb + g.rows_per_cta, g.row0 + g.nrows);
  if (rb >= re) return;
  float* ring = reinterpret_cast<float*>(smem);
  const int nst = (int)((re - rb + g.tr - 1) / g.tr);
  if (tid == 0) {
    for (int s = 0; s < g.ns; ++s) { s_mbar_init(&bars[s], 1); s_mbar_init(&empty[s], ncons); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0 || (producer && lane == 0)) {
    if (tid == 0)
      for (int s = 0; s < nst && s < g.ns; ++s) marg_issue(ring, bars, g, X, rb, re, s);
    if (producer)
      for (int s = g.ns; s < nst; ++s) {   // refill stage s's slot once stage s - ns is released
        s_wait(&empty[s % g.ns], (unsigned)((s / g.ns) - 1) & 1u);
        s_fence_async();
        marg_issue(ring, bars, g, X, rb, re, s);
      }
  }
  long long acc[kMQ][4];
  unsigned acc32[kMQ][4];
#pragma unroll
  for (int m = 0; m < kMQ; ++m)
#pragma unroll
    for (int e = 0; e < 4; ++e) { acc[m][e] = 0; acc32[m][e] = 0u; }
  int steps = 0;
  // MOI 0 with every q of the pass < 2^22 (the store's running max phi and the batch's, read on
  // the device): q = bits(fma(|x|, 2^S, 2^23)) - bits(2^23) exactly (one rounding of the exact
  // value, ties to even), so the biased bits are summed and the bias removed per fold -- one
  // FFMA per element instead of FMUL + F2I (the conversion pipe), mod-2^32 arithmetic exact
  // because every true 32-bit sum is < 2^32
  bool magic = false;
  if (Q32 && MOI == 0) {
    double qm = g.qmax;
    if (g.dphi) qm = fmax(qm, __longlong_as_double((long long)*g.dphi) * scd);
    magic = qm < 4194304.0;
  }
  constexpr unsigned kBias = 0x4B000000u;   // bits(2^23)
  int nvq = 0;                               // this lane's column quads in its chunk
#pragma unroll
  for (int m = 0; m < kMQ; ++m) nvq += 4 * (lane + 32 * m) < cw_real ? 1 : 0;
  const unsigned rbias = magic ? (unsigned)(4 * nvq) * kBias : 0u;   // per row total (mod 2^32)
  long long x3run = 0;   // lane 0: running sum of slice x3k
  int64_t x3k = -1;
  for (int s = 0; s < nst && !producer; ++s) {
    const int64_t r0 = rb + (int64_t)s * g.tr;
    const int nr = (int)min((int64_t)g.tr, re - r0);
    const int slot = s % g.ns;
    s_wait(&bars[slot], (unsigned)(s / g.ns) & 1u);
    const float* st = ring + (size_t)slot * g.tr * g.pitch + c0;
    // (slice, row) of the stage's first row: one division per stage; rows within the stage
    // step from it (a 32-bit division only where a stage wraps past a slice end)
    const int64_t sk0 = r0 / J;
    const int sj0 = (int)(r0 - sk0 * J);
    auto slice_of = [&](int r, int* jo) -> int64_t {
      int jj = sj0 + r;
      int64_t kk = sk0;
      if (jj >= J) { const int q = jj / J; kk += q; jj -= q * J; }
      *jo = jj;
      return kk;
    };
    for (int rw = wslot * kRPW; rw < nr; rw += g.wpc * kRPW) {
      long long rs[kRPW];
      if (Q32) {
        // the two rows of the step together: one IADD3 per column for both rows' values
        static_assert(kRPW == 2, "Q32 path pairs two rows");
        unsigned r32a = 0u, r32b = 0u;
        const bool two = rw + 1 < nr;
        const float* rowa = st + (size_t)rw * g.pitch;
        const float* rowb = rowa + g.pitch;
#pragma unroll
        for (int m = 0; m < kMQ; ++m) {
          const int col = 4 * (lane + 32 * m);
          if (col < cw_real) {
            const float4 xa = *reinterpret_cast<const float4*>(rowa + col);
            const float4 xb = two ? *reinterpret_cast<const float4*>(rowb + col) : make_float4(0.f, 0.f, 0.f, 0.f);
            unsigned a0, a1, a2, a3, b0, b1, b2, b3;
            if (magic) {   // biased: kBias + q
              a0 = __float_as_uint(fmaf(fabsf(xa.x), scf, 8388608.0f));
              a1 = __float_as_uint(fmaf(fabsf(xa.y), scf, 8388608.0f));
              a2 = __float_as_uint(fmaf(fabsf(xa.z), scf, 8388608.0f));
              a3 = __float_as_uint(fmaf(fabsf(xa.w), scf, 8388608.0f));
              b0 = __float_as_uint(fmaf(fabsf(xb.x), scf, 8388608.0f));
              b1 = __float_as_uint(fmaf(fabsf(xb.y), scf, 8388608.0f));
              b2 = __float_as_uint(fmaf(fabsf(xb.z), scf, 8388608.0f));
              b3 = __float_as_uint(fmaf(fabsf(xb.w), scf, 8388608.0f));
            } else {
              a0 = quant32<MOI>(xa.x, scf, scd); a1 = quant32<MOI>(xa.y, scf, scd);
              a2 = quant32<MOI>(xa.z, scf, scd); a3 = quant32<MOI>(xa.w, scf, scd);
              b0 = quant32<MOI>(xb.x, scf, scd); b1 = quant32<MOI>(xb.y, scf, scd);
              b2 = quant32<MOI>(xb.z, scf, scd); b3 = quant32<MOI>(xb.w, scf, scd);
            }
            if (QT && col + 4 > cw_real) {   // QT: I % 4 != 0, a chunk may end inside a quad
              const unsigned z = magic ? kBias : 0u;   // the value of q = 0
              if (col + 1 >= cw_real) { a1 = z; b1 = z; }
              if (col + 2 >= cw_real) { a2 = z; b2 = z; }
              if (col + 3 >= cw_real) { a3 = z; b3 = z; }
            }
            acc32[m][0] += a0 + b0; acc32[m][1] += a1 + b1; acc32[m][2] += a2 + b2; acc32[m][3] += a3 + b3;
            r32a += (a0 + a1) + (a2 + a3);
            r32b += (b0 + b1) + (b2 + b3);
          }
        }
        // exact warp totals of values <= 2^31: 18-bit chunks (sums < 2^23 and 2^19)
        r32a -= rbias;   // a missing second row contributed q = 0 values (xb = 0: biased kBias)
        r32b -= rbias;
        {
          const unsigned lo = __reduce_add_sync(0xffffffffu, r32a & 0x3FFFFu);
          const unsigned hi = __reduce_add_sync(0xffffffffu, r32a >> 18);
          rs[0] = (long long)(((unsigned long long)hi << 18) + lo);
        }
        {
          const unsigned lo = __reduce_add_sync(0xffffffffu, r32b & 0x3FFFFu);
          const unsigned hi = __reduce_add_sync(0xffffffffu, r32b >> 18);
          rs[1] = (long long)(((unsigned long long)hi << 18) + lo);
        }
        if (++steps == g.spill) {
          const unsigned cb = magic ? (unsigned)(2 * steps) * kBias : 0u;   // two biased values per step
          steps = 0;
#pragma unroll
          for (int m = 0; m < kMQ; ++m) {
            const bool vq = 4 * (lane + 32 * m) < cw_real;
#pragma unroll
            for (int e = 0; e < 4; ++e) { acc[m][e] += vq ? acc32[m][e] - cb : 0u; acc32[m][e] = 0u; }
          }
        }
      }
#pragma unroll
      for (int v = 0; v < kRPW; ++v) {
        if (Q32) break;
        rs[v] = 0;
        const int r = rw + v;
        if (r < nr) {
          const float* rowp = st + (size_t)r * g.pitch;
          if (g.dbg == 2) continue;
#pragma unroll
          for (int m = 0; m < kMQ; ++m) {
            const int col = 4 * (lane + 32 * m);
            if (col < cw_real) {
              const float4 x = *reinterpret_cast<const float4*>(rowp + col);
              long long q0, q1, q2, q3;
              if (g.dbg == 1) {
                q0 = __float_as_int(x.x) & 0xffff; q1 = __float_as_int(x.y) & 0xffff;
                q2 = __float_as_int(x.z) & 0xffff; q3 = __float_as_int(x.w) & 0xffff;
              } else {
                q0 = quant<MOI>(x.x, scf, scd); q1 = quant<MOI>(x.y, scf, scd);
                q2 = quant<MOI>(x.z, scf, scd); q3 = quant<MOI>(x.w, scf, scd);
              }
              if (col + 1 >= cw_real) q1 = 0;
              if (col + 2 >= cw_real) q2 = 0;
              if (col + 3 >= cw_real) q3 = 0;
              acc[m][0] += q0; acc[m][1] += q1; acc[m][2] += q2; acc[m][3] += q3;
              rs[v] += (q0 + q1) + (q2 + q3);
            }
          }
        }
      }
      if (!Q32)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int v = 0; v < kRPW; ++v) rs[v] += __shfl_xor_sync(0xffffffffu, rs[v], o);
      // every lane holds the kRPW row totals: lane v adds row v to x2; lane 0 folds them into
      // the warp's running x3 sum of slice x3k (flushed when the slice changes: one global
      // reduction per slice and warp instead of a contended shared 64-bit atomic per row)
      if (lane < kRPW) {
        long long mine = rs[0];
#pragma unroll
        for (int v = 1; v < kRPW; ++v)
          if (lane == v) mine = rs[v];
        const int r = rw + lane;
        if (r < nr && mine) {
          int j;
          slice_of(r, &j);
          atomicAdd(&x2[j], (unsigned long long)mine);
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int v = 0; v < kRPW; ++v) {
          const int r = rw + v;
          if (r < nr) {
            int jdummy;
            const int64_t k = slice_of(r, &jdummy);
            if (k != x3k) {
              if (x3run) atomicAdd(&x3[x3k], (unsigned long long)x3run);
              x3k = k;
              x3run = 0;
            }
            x3run += rs[v];
          }
        }
      }
    }
    if (g.pc) {
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(&empty[slot])) : "memory");
    } else {
      __syncthreads();   // stage consumed by every warp
      if (tid == 0 && s + g.ns < nst) {
        s_fence_async();
        marg_issue(ring, bars, g, X, rb, re, s + g.ns);
      }
    }
  }
  if (lane == 0 && x3run) atomicAdd(&x3[x3k], (unsigned long long)x3run);
  if (Q32) {
    const unsigned cb = magic ? (unsigned)(2 * steps) * kBias : 0u;
#pragma unroll
    for (int m = 0; m < kMQ; ++m) {
      const bool vq = 4 * (lane + 32 * m) < cw_real;
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[m][e] += vq ? acc32[m][e] - cb : 0u;
    }
  }
  // x1: the warps' column sums through the (now idle) ring, summed per column in warp order
  // (every stage has been consumed, so no copy is in flight)
  __syncthreads();
  long long* xw = reinterpret_cast<long long*>(smem);   // [kNW][cw]
#pragma unroll
  for (int m = 0; m < kMQ; ++m)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int col = 4 * (lane + 32 * m) + e;
      if (col < cw_real && warp < g.nch * g.wpc) xw[(size_t)warp * g.cw + col] = acc[m][e];
    }
  __syncthreads();
  for (int c = tid; c < g.ncol; c += blockDim.x) {
    const int ch = c / g.cw, cc = c - ch * g.cw;
    long long t = 0;
    for (int w = ch; w < g.nch * g.wpc; w += g.nch) t += xw[(size_t)w * g.cw + cc];
    if (t) atomicAdd(&x1[c], (unsigned long long)t);
  }
  (void)nwarps;
}

// ---------------------------------------------------------------------------------------
// a7: fit.  inner = sum_{i,j,k} X(i,j,k) m(i,j,k), m = sum_f lam_f A(i,f) B(j,f) C(k,f);
// sq = sum X^2.  Thread t owns the column quad t % NQ of the rows of its row group t / NQ
// and holds lam_f A(i,f) for its 4 columns in registers; W(row,f) = B(j,f) C(k,f) of stage
// s+1 is formed in a double-buffered shared array while stage s is consumed (one barrier per
// stage).  fp32 per element and per stage, fp64 across stages; per-CTA partials reduced in a
// fixed order by fit_combine_kernel.
// ---------------------------------------------------------------------------------------
// a7 fit: inner = <X, [[lam; A, B, C]]> and ||X||^2 in one pass over whole-row stages.  A
// thread owns QPT column quads; row (j, k) needs only B(j, :).  QPT = 1: the thread
// accumulates acc(i, f) += X(i,j,k) B(j,f) over its rows of a slice (independent FMA chains)
// and the slice's lam_f A(i,f) C(k,f) multiplies acc at a fold (slice change, or a stage end
// after >= kFoldRows = 128 rows).  QPT = 2: alc(i,f) = lam_f A(i,f) C(k,f) in registers,
// m(i) = sum_f alc(i,f) B(j,f), inner += X(i,j,k) m(i) (measured faster at 2 quads).  BRES: B (J x RB, zero padded) resident in
// shared memory; else the B rows of stage s+1 are loaded into registers while stage s is
// consumed and stored to a double buffer after it.  fp32 runs, fp64 across folds / stages.
constexpr int kFitT2 = 384;       // fit: threads per CTA at 2 quads per thread (<= 168 registers)

template <int RB, int QPT, bool BRES>
__global__ void __launch_bounds__(QPT == 1 ? kST : kFitT2, 1) fit_stream_kernel(const float* __restrict__ X, StreamGeom g,
                                                            int J, int R, const float* __restrict__ lam,
                                                            const float* __restrict__ A,
                                                            const float* __restrict__ B,
                                                            const float* __restrict__ C,
                                                            double* __restrict__ part,
                                                            const int32_t* __restrict__ kmap) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned long long bars[kMaxNS];
  __shared__ double red[32];
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int nq = g.pitch / 4;
  const int tq = tid % g.tpg, grp = tid / g.tpg;
  const bool active = grp < g.ng;
  const int64_t rb = g.row0 + (int64_t)blockIdx.x * g.rows_per_cta;
  const int64_t re = min(rb + g.rows_per_cta, g.row0 + g.nrows);
  float* ring = reinterpret_cast<float*>(smem);
  float* Wbuf = ring + (size_t)g.ns * g.tr * g.pitch;   // BRES: Bs [J][RB]; else W [2][tr][RB]
  const int nst = rb < re ? (int)((re - rb + g.tr - 1) / g.tr) : 0;
  float wb[kWPT];
  // B rows of the stage starting at row r0 = (j0 of some slice): row r has j = (j0 + r) mod J
  auto load_w = [&](int64_t r0, int j0) {
    const int nr = (int)min((int64_t)g.tr, re - r0);
#pragma unroll
    for (int t = 0; t < kWPT; ++t) {
      const int e = tid + t * nthr;
      wb[t] = 0.f;
      if (e < nr * RB) {
        const int r = e / RB, f = e - r * RB;
        int j = j0 + r;
        if (j >= J) j -= (j / J) * J;
        if (f < R) wb[t] = __ldg(B + (int64_t)j * R + f);
      }
    }
  };
  auto store_w = [&](int s) {
    float* W = Wbuf + (size_t)(s & 1) * g.tr * RB;
#pragma unroll
    for (int t = 0; t < kWPT; ++t) {
      const int e = tid + t * nthr;
      if (e < g.tr * RB) W[e] = wb[t];
    }
  };
  if (tid == 0) {
    for (int s = 0; s < g.ns; ++s) s_mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // stage cursor: slice ks and row js of the first row of the current stage (no divisions
  // in the loop), ring slot and its phase
  int64_t ks = rb / J;
  int js = (int)(rb - ks * J);
  if constexpr (BRES) {
    for (int e = tid; e < J * RB; e += nthr) {
      const int j = e / RB, f = e - j * RB;
      Wbuf[e] = f < R ? B[(int64_t)j * R + f] : 0.f;
    }
  } else {
    if (nst > 0) { load_w(rb, js); store_w(0); }
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < nst && s < g.ns; ++s) marg_issue(ring, bars, g, X, rb, re, s);
  double inner = 0.0, sq = 0.0;
  if constexpr (QPT == 1) {
  // acc(i, f) = sum over the thread's rows (j, k) of one slice k of X(i, j, k) B(j, f) for its
  // QPT column quads: a mode-1 MTTKRP row kept in registers (independent FMA chains); folded
  // into inner += sum_{i,f} lam_f A(i,f) C(k,f) acc(i,f) when the slice changes or at the end
  // of a stage after >= kFoldRows rows (fp32 runs of < kFoldRows + a stage's rows, fp64 across
  // folds).
  constexpr int kFoldRows = 128;
  float acc[QPT][4][RB];
#pragma unroll
  for (int u = 0; u < QPT; ++u)
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int f = 0; f < RB; ++f) acc[u][e][f] = 0.f;
  int64_t kc = -1;
  int run = 0;
  auto fold = [&](int64_t k) {
    const int64_t kg = kmap ? kmap[k] : k;
    float lc[RB];
#pragma unroll
    for (int f = 0; f < RB; ++f) lc[f] = f < R ? lam[f] * C[kg * R + f] : 0.f;
    float t = 0.f;
#pragma unroll
    for (int u = 0; u < QPT; ++u)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 4 * (tq + u * g.tpg) + e;
#pragma unroll
        for (int f = 0; f < RB; ++f) {
          if (i < g.ncol && f < R) t = fmaf(A[(int64_t)i * R + f] * lc[f], acc[u][e][f], t);
          acc[u][e][f] = 0.f;
        }
      }
    inner += (double)t;
    run = 0;
  };
  for (int s = 0; s < nst; ++s) {
    const int slot = s % g.ns;
    const int64_t r0 = rb + (int64_t)s * g.tr;
    const int nr = (int)min((int64_t)g.tr, re - r0);
    int jn = js + g.tr;   // the next stage's first row
    int64_t kn = ks;
    if (jn >= J) { kn += jn / J; jn -= (jn / J) * J; }
    if (!BRES && s + 1 < nst) load_w(r0 + g.tr, jn);   // loads in flight while stage s is consumed
    s_wait(&bars[s % g.ns], (unsigned)(s / g.ns) & 1u);
    if (active) {
      const float* st = ring + (size_t)slot * g.tr * g.pitch;
      const float* W = Wbuf + (BRES ? 0 : (size_t)(s & 1) * g.tr * RB);
      float fs = 0.f;
      // segments of the stage with one slice k each
      int64_t k = ks;   // the stage cursor: (slice, row) of row r0
      int j = js;
      for (int ra = 0; ra < nr;) {
        const int seg = min(nr - ra, J - j);
        if (k != kc) {
          if (kc >= 0) fold(kc);
          kc = k;
        }
#pragma unroll 1
        for (int r = ra + ((grp - ra) % g.ng + g.ng) % g.ng; r < ra + seg; r += g.ng) {
          const float* wr = BRES ? W + (size_t)(j + r - ra) * RB : W + r * RB;
          float w[RB];
          if constexpr (RB % 4 == 0) {
#pragma unroll
            for (int f4 = 0; f4 < RB / 4; ++f4) {
              const float4 wv = *reinterpret_cast<const float4*>(wr + 4 * f4);
              w[4 * f4] = wv.x; w[4 * f4 + 1] = wv.y; w[4 * f4 + 2] = wv.z; w[4 * f4 + 3] = wv.w;
            }
          } else {
#pragma unroll
            for (int f2 = 0; f2 < RB / 2; ++f2) {
              const float2 wv = *reinterpret_cast<const float2*>(wr + 2 * f2);
              w[2 * f2] = wv.x; w[2 * f2 + 1] = wv.y;
            }
          }
#pragma unroll
          for (int u = 0; u < QPT; ++u) {
            const int q = tq + u * g.tpg;
            if (q < nq) {
              const float4 v = *reinterpret_cast<const float4*>(st + (size_t)r * g.pitch + 4 * q);
#pragma unroll
              for (int f = 0; f < RB; ++f) {
                acc[u][0][f] = fmaf(v.x, w[f], acc[u][0][f]);
                acc[u][1][f] = fmaf(v.y, w[f], acc[u][1][f]);
                acc[u][2][f] = fmaf(v.z, w[f], acc[u][2][f]);
                acc[u][3][f] = fmaf(v.w, w[f], acc[u][3][f]);
              }
              // padding columns are zero in the store
              fs = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, fs))));
            }
          }
          ++run;
        }
        ra += seg;
        j = 0;
        ++k;
      }
      if (run >= kFoldRows) fold(kc);   // at stage ends only: the row loop stays branch-free
      sq += (double)fs;
    }
    if (!BRES && s + 1 < nst) store_w(s + 1);   // the other W buffer (free since the last barrier)
    __syncthreads();   // stage (and W(s)) consumed
    if (tid == 0 && s + g.ns < nst) {
      s_fence_async();
      marg_issue(ring, bars, g, X, rb, re, s + g.ns);
    }
    ks = kn;
    js = jn;
  }
  if (active && kc >= 0) fold(kc);
  } else {
  // QPT = 2 (rows of > 2048 floats): the earlier form measures faster there (C4: 30 vs 33 ms)
  // lam_f A(i,f) [* C(k,f) when BRES] of the thread's QPT column quads (tq + u * tpg)
  float al[QPT][4][RB];
  int64_t kc = -1;
  auto load_al = [&](int64_t k) {
    const int64_t kg = kmap ? kmap[k] : k;
#pragma unroll
    for (int u = 0; u < QPT; ++u)
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int f = 0; f < RB; ++f) {
          const int i = 4 * (tq + u * g.tpg) + e;
          float v = 0.f;
          if (active && i < g.ncol && f < R) {
            v = lam[f] * A[(int64_t)i * R + f] * C[kg * R + f];
          }
          al[u][e][f] = v;
        }
  };
  for (int s = 0; s < nst; ++s) {
    const int slot = s % g.ns;
    const int64_t r0 = rb + (int64_t)s * g.tr;
    const int nr = (int)min((int64_t)g.tr, re - r0);
    int jn = js + g.tr;   // the next stage's first row
    int64_t kn = ks;
    if (jn >= J) { kn += jn / J; jn -= (jn / J) * J; }
    if (!BRES && s + 1 < nst) load_w(r0 + g.tr, jn);   // loads in flight while stage s is consumed
    s_wait(&bars[s % g.ns], (unsigned)(s / g.ns) & 1u);
    if (active) {
      const float* st = ring + (size_t)slot * g.tr * g.pitch;
      const float* W = Wbuf + (BRES ? 0 : (size_t)(s & 1) * g.tr * RB);
      float fi = 0.f, fs = 0.f;
      auto rows = [&](int ra, int rb2, int jbase) {   // rows [ra, rb2) of the stage, row r has j = jbase + r - ra
#pragma unroll 1
        for (int r = ra + ((grp - ra) % g.ng + g.ng) % g.ng; r < rb2; r += g.ng) {
          const float* wr = BRES ? W + (size_t)(jbase + r - ra) * RB : W + r * RB;
          float w[RB];
          if constexpr (RB % 4 == 0) {
#pragma unroll
            for (int f4 = 0; f4 < RB / 4; ++f4) {
              const float4 wv = *reinterpret_cast<const float4*>(wr + 4 * f4);
              w[4 * f4] = wv.x; w[4 * f4 + 1] = wv.y; w[4 * f4 + 2] = wv.z; w[4 * f4 + 3] = wv.w;
            }
          } else {
#pragma unroll
            for (int f2 = 0; f2 < RB / 2; ++f2) {
              const float2 wv = *reinterpret_cast<const float2*>(wr + 2 * f2);
              w[2 * f2] = wv.x; w[2 * f2 + 1] = wv.y;
            }
          }
#pragma unroll
          for (int u = 0; u < QPT; ++u) {
            const int q = tq + u * g.tpg;
            if (q < nq) {
              const float4 v = *reinterpret_cast<const float4*>(st + (size_t)r * g.pitch + 4 * q);
              float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
#pragma unroll
              for (int f = 0; f < RB; ++f) {
                m0 = fmaf(al[u][0][f], w[f], m0);
                m1 = fmaf(al[u][1][f], w[f], m1);
                m2 = fmaf(al[u][2][f], w[f], m2);
                m3 = fmaf(al[u][3][f], w[f], m3);
              }
              fi = fmaf(v.x, m0, fmaf(v.y, m1, fmaf(v.z, m2, fmaf(v.w, m3, fi))));
              // padding columns are zero in the store (and carry al == 0)
              fs = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, fs))));
            }
          }
        }
      };
      // segments of the stage with one slice k each; C(k, :) folded into al at a change
      int64_t k = ks;   // the stage cursor: (slice, row) of row r0
      int j = js;
      for (int ra = 0; ra < nr;) {
        const int seg = min(nr - ra, J - j);
        if (k != kc) {
          inner += (double)fi;
          fi = 0.f;
          load_al(k);
          kc = k;
        }
        rows(ra, ra + seg, j);
        ra += seg;
        j = 0;
        ++k;
      }
      inner += (double)fi;
      sq += (double)fs;
    }
    if (!BRES && s + 1 < nst) store_w(s + 1);   // the other W buffer (free since the last barrier)
    __syncthreads();   // stage (and W(s)) consumed
    if (tid == 0 && s + g.ns < nst) {
      s_fence_async();
      marg_issue(ring, bars, g, X, rb, re, s + g.ns);
    }
    ks = kn;
    js = jn;
  }
  }
  inner = block_sum_d(inner, red);
  sq = block_sum_d(sq, red);
  if (tid == 0) {
    part[2 * blockIdx.x] = inner;
    part[2 * blockIdx.x + 1] = sq;
  }
}

// The block stages the partials and Grams in shared memory with coalesced loads; thread 0 then
// sums them in the fixed sequential order (no global-load latency chain).
constexpr int kCombT = 256;
__global__ void __launch_bounds__(kCombT) fit_combine_kernel(const double* part, int nb, const double* G,
                                                            const float* lam, int R, double* relerr) {
  __shared__ double sp[2 * kNumSMs];
  __shared__ double sg[3 * kMaxR * kMaxR];
  __shared__ double sl[kMaxR];
  for (int e = threadIdx.x; e < 2 * nb; e += blockDim.x) sp[e] = part[e];
  for (int e = threadIdx.x; e < 3 * R * R; e += blockDim.x) sg[e] = G[e];
  for (int e = threadIdx.x; e < R; e += blockDim.x) sl[e] = (double)lam[e];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double inner = 0.0, sq = 0.0, mn = 0.0;
  for (int b = 0; b < nb; ++b) { inner += sp[2 * b]; sq += sp[2 * b + 1]; }
  for (int f = 0; f < R; ++f)
    for (int g = 0; g < R; ++g)
      mn += sl[f] * sl[g] * sg[f * R + g] * sg[R * R + f * R + g] * sg[2 * R * R + f * R + g];
  const double res = fmax(0.0, sq - 2.0 * inner + mn);
  *relerr = sq > 0.0 ? sqrt(res / sq) : 0.0;
}

constexpr int kRingBytes = 192 * 1024;

// Marginal pass: stages of whole rows (one bulk copy each, contiguous in the store); a row is
// split into nch chunks of <= 512 floats, each worked by wpc warps (nch * wpc <= 16); rows per
// stage a multiple of kRPW * wpc, two ~96 KB stages in a 192 KB ring.
StreamGeom marg_geom(const DenseView& X, int64_t k0, int64_t nk, int* gx, int* gy, int* threads) {
  StreamGeom g{};
  g.row0 = k0 * X.J;
  g.nrows = nk * X.J;
  g.pitch = (int)X.pitch;
  g.ncol = (int)X.I;
  const int maxcw = 4 * 32 * kMQ;
  g.nch = (g.pitch + maxcw - 1) / maxcw;
  // chunks per row rounded up to a divisor of the CTA's warps, so every warp has a chunk (C4: 6 -> 8
  // chunks of 376 floats, 16 warps; measured ~2 % faster than 12 warps on 500-float chunks)
  while (g.nch < kNW && kNW % g.nch) ++g.nch;
  static const int nch_env = getenv("SBT_MARG_NCH") ? atoi(getenv("SBT_MARG_NCH")) : 0;
  if (nch_env > g.nch && nch_env <= kNW) g.nch = nch_env;   // narrower chunks (tuning experiment)
  g.cw = ((g.pitch + g.nch - 1) / g.nch + 3) & ~3;
  g.wpc = kNW / g.nch;
  if (g.wpc < 1) g.wpc = 1;
  const int unit = kRPW * g.wpc;
  const int row_b = g.pitch * (int)sizeof(float);
  // stage / ring sizes (SBT_MARG_STAGE_KB / SBT_MARG_RING_KB: tuning experiments)
  static const int stage_kb = getenv("SBT_MARG_STAGE_KB") ? atoi(getenv("SBT_MARG_STAGE_KB")) : 96;
  static const int ring_kb = getenv("SBT_MARG_RING_KB") ? atoi(getenv("SBT_MARG_RING_KB")) : 192;
  int m = (stage_kb * 1024) / (unit * row_b);   // ~96 KB stages: two in the ring (fewer barriers)
  if (m < 1) m = 1;
  g.tr = unit * m;
  g.ns = ring_kb * 1024 / (g.tr * row_b);
  if (g.ns > kMaxNS) g.ns = kMaxNS;
  if (g.ns < 2) { g.ns = 2; }
  int64_t nx = (int64_t)kNumSMs * kMargCTAs;
  if (nx > ceil_div(g.nrows, 2 * g.tr)) nx = ceil_div(g.nrows, 2 * g.tr);
  if (nx < 1) nx = 1;
  g.rows_per_cta = ceil_div(g.nrows, nx);
  *gx = (int)ceil_div(g.nrows, g.rows_per_cta);
  *gy = 1;
  static const int pc = getenv("SBT_MARG_PC") ? atoi(getenv("SBT_MARG_PC")) : 0;
  static const int dbg = getenv("SBT_MARG_DBG") ? atoi(getenv("SBT_MARG_DBG")) : 0;
  g.dbg = dbg;
  g.pc = pc && g.nch * g.wpc < kNW;   // room for the producer warp
  *threads = 32 * (g.nch * g.wpc + (g.pc ? 1 : 0));
  return g;
}
// Fit pass: stages of whole rows (one bulk copy); thread (group grp, lane tq) owns the column
// quads tq + u * tpg (u < qpt) and the rows grp, grp + ng, ... of each stage; stages of ~32 KB.
StreamGeom fit_geom(const DenseView& X, int RB, int* gx, int* gy, int* threads) {
  StreamGeom g{};
  g.row0 = 0;
  g.nrows = X.J * X.K;
  g.pitch = (int)X.pitch;
  g.ncol = (int)X.I;
  const int nq = g.pitch / 4;
  g.qpt = nq <= kST ? 1 : 2;   // 2: nq <= 2 * kFitT2 (fit_stream_supported)
  g.tpg = (nq + g.qpt - 1) / g.qpt;
  const int tmax = g.qpt == 1 ? kST : kFitT2;
  g.ng = tmax / g.tpg > 0 ? tmax / g.tpg : 1;
  int nthr = ((g.ng * g.tpg + 31) / 32) * 32;
  if (nthr > tmax) nthr = tmax;
  const int row_b = g.pitch * (int)sizeof(float);
  const size_t bres_b = sizeof(float) * (size_t)X.J * RB;
  g.bres = bres_b <= 48 * 1024;
  g.tr = (96 * 1024) / row_b;   // ~96 KB stages: two in the ring (one barrier per stage)
  if (g.tr < 1) g.tr = 1;
  if (!g.bres && g.tr * RB > kWPT * nthr) g.tr = kWPT * nthr / RB;   // the B prefetch registers
  if (g.tr > 256) g.tr = 256;
  const size_t extra = g.bres ? bres_b : sizeof(float) * 2 * (size_t)g.tr * RB;
  const int ring_b = (int)(208 * 1024 - extra);
  g.cw = g.pitch;
  g.ns = ring_b / (g.tr * row_b);
  if (g.ns > kMaxNS) g.ns = kMaxNS;
  if (g.ns < 2) {   // very long rows: two stages of fewer rows
    g.ns = 2;
    g.tr = std::max(1, ring_b / (2 * row_b));
  }
  int64_t nx = kNumSMs;
  if (nx > ceil_div(g.nrows, 2 * g.tr)) nx = ceil_div(g.nrows, 2 * g.tr);
  if (nx < 1) nx = 1;
  g.rows_per_cta = ceil_div(g.nrows, nx);
  *gx = (int)ceil_div(g.nrows, g.rows_per_cta);
  *gy = 1;
  *threads = nthr;
  return g;
}


// ---------------------------------------------------------------------------------------
// a1 + lag-1 a7 in ONE pass (second half; Alg. 1 l.2 and
// P:409-413): while update t+1 streams the old slices [0, K_t) for its marginals, the same
// bytes give <X_t, [[lam; A, B, C]]_t> and ||X_t||^2 of the model update t committed (its C
// has exactly the rows of those slices).  Thread layout of the fit pass with the row groups
// padded to whole warps (a warp never straddles two rows): thread (group grp, lane tq) owns
// the column quads tq + u * tpg of rows grp, grp + ng, ...; per element: the fit's FMAs (as
// fit_stream_kernel), fp32 sum of squares, and q(x) = RNE(phi(x) 2^S) added to the thread's
// int64 column sums (x1) and to its row partial, reduced over the warp per row (butterfly)
// -> one global atomic per row and warp (x2) and a per-warp running sum per slice (x3), as
// marg_stream_kernel.  Integer marginals: bit-identical to the separate pass.
// ---------------------------------------------------------------------------------------
// Exact warp sum of non-negative 64-bit values by 21-bit chunks through the warp-reduce unit
// (REDUX: one instruction per chunk, no shuffle tree): each chunk's 32-lane sum is < 2^26.
// NCH = 2 covers values < 2^42, NCH = 3 values < 2^63.
template <int NCH>
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
  unsigned long long t = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const unsigned part = (unsigned)(v >> (21 * c)) & 0x1FFFFFu;
    t += (unsigned long long)__reduce_add_sync(0xffffffffu, part) << (21 * c);
  }
  return t;
}

template <int MOI, int RB, int QPT, bool BRES, bool Q32>
__global__ void __launch_bounds__(QPT == 1 ? kST : kFitT2, 1) margfit_stream_kernel(
    const float* __restrict__ X, StreamGeom g, int J, int R, float scf, double scd,
    const float* __restrict__ lam, const float* __restrict__ A, const float* __restrict__ B,
    const float* __restrict__ C, double* __restrict__ part, unsigned long long* __restrict__ x1,
    unsigned long long* __restrict__ x2, unsigned long long* __restrict__ x3, const int32_t* __restrict__ kmap) {
  // Q32 (plan-time guarantee on q <= 2^qb): 32-bit quantised values, row partials and per-stage
  // column sums (folded into 64-bit column sums at stage ends); else 64-bit throughout.
  // Shared memory is addressed by byte offsets from the extern array (32-bit LDS addressing;
  // no generic-pointer window arithmetic in the row loop).
  using qint = typename std::conditional<Q32, unsigned, unsigned long long>::type;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned long long bars[kMaxNS];
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, nthr = blockDim.x;
  const int nq = g.pitch / 4;
  const int tq = tid % g.tpg, grp = tid / g.tpg;   // g.tpg: a multiple of 32
  const bool active = grp < g.ng;
  const int ng = g.ng;
  const int64_t rb = g.row0 + (int64_t)blockIdx.x * g.rows_per_cta;
  const int64_t re = min(rb + g.rows_per_cta, g.row0 + g.nrows);
  const int pitchB = g.pitch * (int)sizeof(float);
  const int stageB = g.tr * pitchB;
  float* Wbuf = reinterpret_cast<float*>(smem + (size_t)g.ns * stageB);   // BRES: Bs [J][RB]; else W [2][tr][RB]
  const int nst = rb < re ? (int)((re - rb + g.tr - 1) / g.tr) : 0;
  // the warp's largest column quad decides whether every lane's quads are real columns
  const int wq_max = (tid | 31) % g.tpg;
  const bool wfull = QPT == 1 ? wq_max < nq : wq_max + g.tpg < nq;
  const bool q1ok = QPT == 2 && tq + g.tpg < nq;
  float wb[kWPT];
  auto load_w = [&](int64_t r0, int j0) {
    const int nr = (int)min((int64_t)g.tr, re - r0);
#pragma unroll
    for (int t = 0; t < kWPT; ++t) {
      const int e = tid + t * nthr;
      wb[t] = 0.f;
      if (e < nr * RB) {
        const int r = e / RB, f = e - r * RB;
        int j = j0 + r;
        if (j >= J) j -= (j / J) * J;
        if (f < R) wb[t] = __ldg(B + (int64_t)j * R + f);
      }
    }
  };
  auto store_w = [&](int s) {
    float* W = Wbuf + (size_t)(s & 1) * g.tr * RB;
#pragma unroll
    for (int t = 0; t < kWPT; ++t) {
      const int e = tid + t * nthr;
      if (e < g.tr * RB) W[e] = wb[t];
    }
  };
  if (tid == 0) {
    for (int s = 0; s < g.ns; ++s) s_mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  int64_t ks = rb / J;
  int js = (int)(rb - ks * J);
  if constexpr (BRES) {
    for (int e = tid; e < J * RB; e += nthr) {
      const int j = e / RB, f = e - j * RB;
      Wbuf[e] = f < R ? B[(int64_t)j * R + f] : 0.f;
    }
  } else {
    if (nst > 0) { load_w(rb, js); store_w(0); }
  }
  __syncthreads();
  float* ring = reinterpret_cast<float*>(smem);
  if (tid == 0)
    for (int s = 0; s < nst && s < g.ns; ++s) marg_issue(ring, bars, g, X, rb, re, s);
  double inner = 0.0, sq = 0.0;
  // x1 column sums of the thread's quads: 64-bit totals in shared memory (registers are the
  // scarce resource here), this stage's sums in registers, folded at every stage end
  const size_t wbytes = BRES ? sizeof(float) * (size_t)J * RB : sizeof(float) * 2 * (size_t)g.tr * RB;
  unsigned long long* xsm = reinterpret_cast<unsigned long long*>(smem + (((size_t)g.ns * stageB + wbytes + 15) & ~(size_t)15));
  qint xs[QPT][4];
#pragma unroll
  for (int u = 0; u < QPT; ++u)
#pragma unroll
    for (int e = 0; e < 4; ++e) { xsm[(u * 4 + e) * nthr + tid] = 0; xs[u][e] = 0; }
  unsigned long long x3acc = 0;    // the lane's share of slice x3k (flushed at slice changes)
  int64_t x3k = -1;
  auto flush_x3 = [&]() {
    const unsigned long long t = warp_sum_u64<3>(x3acc);
    if (lane == 0 && t) atomicAdd(&x3[x3k], t);
    x3acc = 0;
  };
  auto row_x2 = [&](qint rs, int j) {   // the warp's share of row (j, k) -> x2[j]
    unsigned long long t;
    if constexpr (Q32) t = warp_sum_u31(rs);
    else t = warp_sum_u64<3>(rs);
    if (lane == 0 && t) atomicAdd(&x2[j], t);
    x3acc += rs;
  };
  auto quad_marg = [&](const float4& v, qint (&xq)[4]) -> qint {
    qint q0, q1, q2, q3;
    if constexpr (Q32) {
      q0 = quant32<MOI>(v.x, scf, scd); q1 = quant32<MOI>(v.y, scf, scd);
      q2 = quant32<MOI>(v.z, scf, scd); q3 = quant32<MOI>(v.w, scf, scd);
    } else {
      q0 = (qint)quant<MOI>(v.x, scf, scd); q1 = (qint)quant<MOI>(v.y, scf, scd);
      q2 = (qint)quant<MOI>(v.z, scf, scd); q3 = (qint)quant<MOI>(v.w, scf, scd);
    }
    xq[0] += q0; xq[1] += q1; xq[2] += q2; xq[3] += q3;
    return (q0 + q1) + (q2 + q3);   // padding columns are zero in the store: q = 0
  };
  auto fold_x1 = [&]() {
#pragma unroll
    for (int u = 0; u < QPT; ++u)
#pragma unroll
      for (int e = 0; e < 4; ++e) { xsm[(u * 4 + e) * nthr + tid] += xs[u][e]; xs[u][e] = 0; }
  };
  auto wrow = [&](const float* wr, float (&w)[RB]) {
    if constexpr (RB % 4 == 0) {
#pragma unroll
      for (int f4 = 0; f4 < RB / 4; ++f4) {
        const float4 wv = *reinterpret_cast<const float4*>(wr + 4 * f4);
        w[4 * f4] = wv.x; w[4 * f4 + 1] = wv.y; w[4 * f4 + 2] = wv.z; w[4 * f4 + 3] = wv.w;
      }
    } else {
#pragma unroll
      for (int f2 = 0; f2 < RB / 2; ++f2) {
        const float2 wv = *reinterpret_cast<const float2*>(wr + 2 * f2);
        w[2 * f2] = wv.x; w[2 * f2 + 1] = wv.y;
      }
    }
  };
  auto ldv = [&](int off) -> float4 { return *reinterpret_cast<const float4*>(smem + off); };
  if constexpr (QPT == 1) {
    constexpr int kFoldRows = 128;
    float acc[4][RB];
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int f = 0; f < RB; ++f) acc[e][f] = 0.f;
    int64_t kc = -1;
    int run = 0;
    auto fold = [&](int64_t k) {
      const int64_t kg = kmap ? kmap[k] : k;   // sharded store: local slice -> model row
      float lc[RB];
#pragma unroll
      for (int f = 0; f < RB; ++f) lc[f] = f < R ? lam[f] * C[kg * R + f] : 0.f;
      float t = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 4 * tq + e;
#pragma unroll
        for (int f = 0; f < RB; ++f) {
          if (i < g.ncol && f < R) t = fmaf(A[(int64_t)i * R + f] * lc[f], acc[e][f], t);
          acc[e][f] = 0.f;
        }
      }
      inner += (double)t;
      run = 0;
    };
    for (int s = 0; s < nst; ++s) {
      const int slot = s % g.ns;
      const int64_t r0 = rb + (int64_t)s * g.tr;
      const int nr = (int)min((int64_t)g.tr, re - r0);
      int jn = js + g.tr;
      int64_t kn = ks;
      if (jn >= J) { kn += jn / J; jn -= (jn / J) * J; }
      if (!BRES && s + 1 < nst) load_w(r0 + g.tr, jn);
      s_wait(&bars[slot], (unsigned)(s / g.ns) & 1u);
      if (active) {
        const int soff = slot * stageB + 16 * tq;
        const float* W = Wbuf + (BRES ? 0 : (size_t)(s & 1) * g.tr * RB);
        float fs = 0.f;
        int64_t k = ks;
        int j = js;
        for (int ra = 0; ra < nr;) {
          const int seg = min(nr - ra, J - j);
          if (k != kc) {
            if (kc >= 0) fold(kc);
            kc = k;
          }
          if (k != x3k) {
            if (x3k >= 0) flush_x3();
            x3k = k;
          }
          auto rows = [&](auto fullc) {
            constexpr bool FULL = decltype(fullc)::value;
#pragma unroll 1
            for (int r = ra + ((grp - ra) % ng + ng) % ng; r < ra + seg; r += ng) {
              const float* wr = BRES ? W + (size_t)(j + r - ra) * RB : W + r * RB;
              qint rs = 0;
              if (FULL || tq < nq) {
                float w[RB];
                wrow(wr, w);
                const float4 v = ldv(soff + r * pitchB);
#pragma unroll
                for (int f = 0; f < RB; ++f) {
                  acc[0][f] = fmaf(v.x, w[f], acc[0][f]);
                  acc[1][f] = fmaf(v.y, w[f], acc[1][f]);
                  acc[2][f] = fmaf(v.z, w[f], acc[2][f]);
                  acc[3][f] = fmaf(v.w, w[f], acc[3][f]);
                }
                fs = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, fs))));
                rs = quad_marg(v, xs[0]);
              }
              row_x2(rs, j + r - ra);
            }
          };
          if (wfull) rows(std::true_type{});
          else rows(std::false_type{});
          run += (seg + ng - 1) / ng;
          ra += seg;
          j = 0;
          ++k;
        }
        if (run >= kFoldRows) fold(kc);
        sq += (double)fs;
        fold_x1();
      }
      if (!BRES && s + 1 < nst) store_w(s + 1);
      __syncthreads();
      if (tid == 0 && s + g.ns < nst) {
        s_fence_async();
        marg_issue(ring, bars, g, X, rb, re, s + g.ns);
      }
      ks = kn;
      js = jn;
    }
    if (active && kc >= 0) fold(kc);
  } else {
    float al[QPT][4][RB];
    int64_t kc = -1;
    auto load_al = [&](int64_t k) {
      const int64_t kg = kmap ? kmap[k] : k;
#pragma unroll
      for (int u = 0; u < QPT; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int f = 0; f < RB; ++f) {
            const int i = 4 * (tq + u * g.tpg) + e;
            float v = 0.f;
            if (active && i < g.ncol && f < R) v = lam[f] * A[(int64_t)i * R + f] * C[kg * R + f];
            al[u][e][f] = v;
          }
    };
    const int uoff = 16 * g.tpg;   // byte offset of the thread's second quad
    for (int s = 0; s < nst; ++s) {
      const int slot = s % g.ns;
      const int64_t r0 = rb + (int64_t)s * g.tr;
      const int nr = (int)min((int64_t)g.tr, re - r0);
      int jn = js + g.tr;
      int64_t kn = ks;
      if (jn >= J) { kn += jn / J; jn -= (jn / J) * J; }
      if (!BRES && s + 1 < nst) load_w(r0 + g.tr, jn);
      s_wait(&bars[slot], (unsigned)(s / g.ns) & 1u);
      if (active) {
        const int soff = slot * stageB + 16 * tq;
        const float* W = Wbuf + (BRES ? 0 : (size_t)(s & 1) * g.tr * RB);
        float fi = 0.f, fs = 0.f;
        int64_t k = ks;
        int j = js;
        for (int ra = 0; ra < nr;) {
          const int seg = min(nr - ra, J - j);
          if (k != kc) {
            inner += (double)fi;
            fi = 0.f;
            load_al(k);
            kc = k;
          }
          if (k != x3k) {
            if (x3k >= 0) flush_x3();
            x3k = k;
          }
          auto rows = [&](auto fullc) {
            constexpr bool FULL = decltype(fullc)::value;
#pragma unroll 1
            for (int r = ra + ((grp - ra) % ng + ng) % ng; r < ra + seg; r += ng) {
              const float* wr = BRES ? W + (size_t)(j + r - ra) * RB : W + r * RB;
              float w[RB];
              wrow(wr, w);
              const int off = soff + r * pitchB;
              qint rs;
              {
                const float4 v = ldv(off);
                float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
#pragma unroll
                for (int f = 0; f < RB; ++f) {
                  m0 = fmaf(al[0][0][f], w[f], m0);
                  m1 = fmaf(al[0][1][f], w[f], m1);
                  m2 = fmaf(al[0][2][f], w[f], m2);
                  m3 = fmaf(al[0][3][f], w[f], m3);
                }
                fi = fmaf(v.x, m0, fmaf(v.y, m1, fmaf(v.z, m2, fmaf(v.w, m3, fi))));
                fs = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, fs))));
                rs = quad_marg(v, xs[0]);
              }
              {
                // the second quad: a lane past the last column reads its first quad again and
                // contributes zeros (its al columns are zero too) -- no branch in the loop
                float4 v = ldv(q1ok ? off + uoff : off);
                if (!q1ok) v = make_float4(0.f, 0.f, 0.f, 0.f);
                float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
#pragma unroll
                for (int f = 0; f < RB; ++f) {
                  m0 = fmaf(al[1][0][f], w[f], m0);
                  m1 = fmaf(al[1][1][f], w[f], m1);
                  m2 = fmaf(al[1][2][f], w[f], m2);
                  m3 = fmaf(al[1][3][f], w[f], m3);
                }
                fi = fmaf(v.x, m0, fmaf(v.y, m1, fmaf(v.z, m2, fmaf(v.w, m3, fi))));
                fs = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, fs))));
                rs += quad_marg(v, xs[1]);
              }
              row_x2(rs, j + r - ra);
            }
          };
          rows(std::true_type{});
          ra += seg;
          j = 0;
          ++k;
        }
        inner += (double)fi;
        sq += (double)fs;
        fold_x1();
      }
      if (!BRES && s + 1 < nst) store_w(s + 1);
      __syncthreads();
      if (tid == 0 && s + g.ns < nst) {
        s_fence_async();
        marg_issue(ring, bars, g, X, rb, re, s + g.ns);
      }
      ks = kn;
      js = jn;
    }
  }
  if (active && x3k >= 0) flush_x3();
  inner = block_sum_d(inner, red);
  sq = block_sum_d(sq, red);
  if (tid == 0) {
    part[2 * blockIdx.x] = inner;
    part[2 * blockIdx.x + 1] = sq;
  }
  // x1: the groups' column sums through the (idle) ring, summed per column in group order
  __syncthreads();
  unsigned long long* xg = reinterpret_cast<unsigned long long*>(smem);   // [ng][pitch]
  if (active)
#pragma unroll
    for (int u = 0; u < QPT; ++u)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int q = tq + u * g.tpg;
        if (q < nq) xg[(size_t)grp * g.pitch + 4 * q + e] = xsm[(u * 4 + e) * nthr + tid];
      }
  __syncthreads();
  for (int c = tid; c < g.ncol; c += nthr) {
    unsigned long long t = 0;
    for (int gi = 0; gi < g.ng; ++gi) t += xg[(size_t)gi * g.pitch + c];
    if (t) atomicAdd(&x1[c], t);
  }
}

// Fused pass geometry: the fit's, with the row groups padded to whole warps.
StreamGeom margfit_geom(const DenseView& X, int64_t k0, int64_t nk, int RB, int* gx, int* threads) {
  StreamGeom g{};
  g.row0 = k0 * X.J;
  g.nrows = nk * X.J;
  g.pitch = (int)X.pitch;
  g.ncol = (int)X.I;
  const int nq = g.pitch / 4;
  g.qpt = nq <= kST ? 1 : 2;
  const int tpg = (nq + g.qpt - 1) / g.qpt;
  g.tpg = (tpg + 31) & ~31;
  const int tmax = g.qpt == 1 ? kST : kFitT2;
  g.ng = tmax / g.tpg > 0 ? tmax / g.tpg : 1;
  const int nthr = g.ng * g.tpg;
  const int row_b = g.pitch * (int)sizeof(float);
  const size_t bres_b = sizeof(float) * (size_t)X.J * RB;
  g.bres = bres_b <= 48 * 1024;
  g.tr = (96 * 1024) / row_b;
  if (g.tr < 1) g.tr = 1;
  if (!g.bres && g.tr * RB > kWPT * nthr) g.tr = kWPT * nthr / RB;
  if (g.tr > 256) g.tr = 256;
  const size_t extra = (g.bres ? bres_b : sizeof(float) * 2 * (size_t)g.tr * RB) + 16 +
                       sizeof(unsigned long long) * 4 * g.qpt * nthr;   // + the x1 totals
  const int ring_b = (int)(220 * 1024 - extra);
  g.cw = g.pitch;
  g.ns = ring_b / (g.tr * row_b);
  if (g.ns > kMaxNS) g.ns = kMaxNS;
  if (g.ns < 2) {
    g.ns = 2;
    g.tr = std::max(1, ring_b / (2 * row_b));
  }
  int64_t nx = kNumSMs;
  if (nx > ceil_div(g.nrows, 2 * g.tr)) nx = ceil_div(g.nrows, 2 * g.tr);
  if (nx < 1) nx = 1;
  g.rows_per_cta = ceil_div(g.nrows, nx);
  *gx = (int)ceil_div(g.nrows, g.rows_per_cta);
  *threads = nthr;
  return g;
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

// the fit pass additionally needs its quads in registers: <= 2 per thread, and R <= 12 at 2
bool fit_stream_supported(const DenseView& X, int R) {
  if (!stream_supported(X) || R > 16) return false;
  const int nq = (int)(X.pitch / 4);
  return nq <= kST || (nq <= 2 * kFitT2 && R <= 12);
}

bool stream_supported(const DenseView& X) {
  return X.pitch % 4 == 0 && ((uintptr_t)X.base & 15) == 0 && X.I >= 1 && X.I <= 8192 && X.J >= 1;
}

cudaError_t launch_marginals_stream(const DenseView& X, int64_t k0, int64_t nk, int moi, int S,
                                    int64_t* x1, int64_t* x2, int64_t* x3, cudaStream_t st, int qb,
                                    double phimax, const unsigned long long* d_phimax) {
  if (nk <= 0) return cudaSuccess;
  int gx, gy, nthr;
  StreamGeom g = marg_geom(X, k0, nk, &gx, &gy, &nthr);
  // SBT_MARG_FORCE_QB (profiling hook for the small C4 stand-ins, whose capacity bound is 29 bits
  // but whose data stay far below 2^27): the kernel instantiation C4 runs
  if (const char* f = getenv("SBT_MARG_FORCE_QB")) qb = atoi(f);
  const bool q32 = qb <= 27 && !getenv("SAMBATEN_MARG_NO_Q32");
  g.spill = q32 ? (int)(0xFFFFFFFFull / ((unsigned long long)kRPW << qb)) : 0;   // >= 15
  g.qmax = phimax * ldexp(1.0, S);   // phimax: upper bound on phi of the pass (inf: unknown)
  g.dphi = d_phimax;
  if (getenv("SAMBATEN_MARG_NO_MAGIC")) g.qmax = 1e300, g.dphi = nullptr;
  const float scf = ldexpf(1.0f, S < -126 ? -126 : (S > 127 ? 127 : S));
  const double scd = ldexp(1.0, S);
  const size_t smem = sizeof(float) * (size_t)g.ns * g.tr * g.pitch;
  auto* u1 = reinterpret_cast<unsigned long long*>(x1);
  auto* u2 = reinterpret_cast<unsigned long long*>(x2);
  auto* u3 = reinterpret_cast<unsigned long long*>(x3);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<dim3(gx, gy), nthr, smem, st>>>(X.base, g, (int)X.J, scf, scd, u1, u2, u3);
  };
  const bool qt = X.I % 4 != 0;   // chunks are multiples of 4 floats: only the last can end mid-quad
  if (moi == 0) q32 ? (qt ? go(marg_stream_kernel<0, true, true>) : go(marg_stream_kernel<0, true, false>))
                    : go(marg_stream_kernel<0, false>);
  else q32 ? (qt ? go(marg_stream_kernel<1, true, true>) : go(marg_stream_kernel<1, true, false>))
           : go(marg_stream_kernel<1, false>);
  return cudaGetLastError();
}

size_t fit_stream_ws_doubles(const DenseView& X) {   // <= kNumSMs CTA partials
  return 2 * (size_t)kNumSMs + 3 * kMaxR * kMaxR + 8 + gram3_ws_doubles(X.I, X.J, X.K, kMaxR);
}

template <int RB, int QPT, bool BRES>
static cudaError_t fit_go(const DenseView& X, const StreamGeom& g, int gx, int nt, size_t smem, int R,
                          const float* lam, const float* A, const float* B, const float* C, double* part,
                          const int32_t* kmap, cudaStream_t st) {
  cudaFuncSetAttribute(fit_stream_kernel<RB, QPT, BRES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fit_stream_kernel<RB, QPT, BRES><<<gx, nt, smem, st>>>(X.base, g, (int)X.J, R, lam, A, B, C, part, kmap);
  return cudaGetLastError();
}

// one fit pass (per-CTA partials in part[2 * gx]); QPT from the geometry
template <int RB>
static cudaError_t fit_pass(const DenseView& X, const float* lam, const float* A, const float* B, const float* C,
                            int R, const int32_t* kmap, double* part, int* nparts, cudaStream_t st) {
  int gx, gy, nt;
  StreamGeom g = fit_geom(X, RB, &gx, &gy, &nt);
  const size_t extra = g.bres ? (size_t)X.J * RB : 2 * (size_t)g.tr * RB;
  const size_t smem = sizeof(float) * ((size_t)g.ns * g.tr * g.pitch + extra);
  *nparts = gx;
  if (g.qpt == 1) {
    if (g.bres) return fit_go<RB, 1, true>(X, g, gx, nt, smem, R, lam, A, B, C, part, kmap, st);
    return fit_go<RB, 1, false>(X, g, gx, nt, smem, R, lam, A, B, C, part, kmap, st);
  }
  if constexpr (RB <= 12) {
    if (g.bres) return fit_go<RB, 2, true>(X, g, gx, nt, smem, R, lam, A, B, C, part, kmap, st);
    return fit_go<RB, 2, false>(X, g, gx, nt, smem, R, lam, A, B, C, part, kmap, st);
  } else {
    return cudaErrorInvalidValue;   // excluded by fit_stream_supported
  }
}

template <int RB>
static cudaError_t fit_stream_rb(const DenseView& X, const float* lam, const float* A, const float* B,
                                 const float* C, int R, double* ws, double* relerr, cudaStream_t st) {
  double* part = ws;
  int nparts = 0;
  cudaError_t e = fit_pass<RB>(X, lam, A, B, C, R, nullptr, part, &nparts, st);
  if (e != cudaSuccess) return e;
  double* G = ws + 2 * (size_t)kNumSMs;
  e = launch_gram3(A, B, C, X.I, X.J, X.K, R, G, G + 3 * kMaxR * kMaxR, st);
  if (e != cudaSuccess) return e;
  fit_combine_kernel<<<1, kCombT, 0, st>>>(part, nparts, G, lam, R, relerr);
  return cudaGetLastError();
}

__global__ void sum_pairs_kernel(const double* part, int nb, double* out2) {
  if (threadIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int i = 0; i < nb; ++i) { a += part[2 * i]; b += part[2 * i + 1]; }
  out2[0] = a;
  out2[1] = b;
}

// ---- a1 + lag-1 fit: one pass over slices [0, nk) ----------------------------------------------
template <int RB, int MOI>
static cudaError_t margfit_rb(const DenseView& X, int64_t nk, int S, int qb, const float* lam, const float* A,
                              const float* B, const float* C, int R, const int32_t* kmap, int64_t* x1,
                              int64_t* x2, int64_t* x3, double* ws, double* out2, cudaStream_t st) {
  int gx, nt;
  StreamGeom g = margfit_geom(X, 0, nk, RB, &gx, &nt);
  const size_t extra = g.bres ? (size_t)X.J * RB : 2 * (size_t)g.tr * RB;
  size_t smem = ((sizeof(float) * ((size_t)g.ns * g.tr * g.pitch + extra) + 15) & ~(size_t)15) +
                sizeof(unsigned long long) * 4 * g.qpt * nt;
  const size_t xg = sizeof(long long) * (size_t)g.ng * g.pitch;   // x1 combine reuses the ring
  if ((size_t)g.ns * g.tr * g.pitch * sizeof(float) < xg) return cudaErrorInvalidValue;
  const float scf = ldexpf(1.0f, S < -126 ? -126 : (S > 127 ? 127 : S));
  const double scd = ldexp(1.0, S);
  auto* u1 = reinterpret_cast<unsigned long long*>(x1);
  auto* u2 = reinterpret_cast<unsigned long long*>(x2);
  auto* u3 = reinterpret_cast<unsigned long long*>(x3);
  double* part = ws;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<gx, nt, smem, st>>>(X.base, g, (int)X.J, R, scf, scd, lam, A, B, C, part, u1, u2, u3, kmap);
  };
  // 32-bit marginal arithmetic when every q <= 2^qb keeps a lane's row partial (4 QPT values)
  // and its per-stage column sums (<= ceil(tr / ng) rows) below 2^32
  int rows_bits = 0;
  while ((1 << rows_bits) < (g.tr + g.ng - 1) / g.ng) ++rows_bits;
  const bool q32 = qb + std::max(g.qpt == 2 ? 3 : 2, rows_bits) <= 31 && (MOI == 0 || qb <= 31);
  if (g.qpt == 1) {
    if (q32) { if (g.bres) go(margfit_stream_kernel<MOI, RB, 1, true, true>); else go(margfit_stream_kernel<MOI, RB, 1, false, true>); }
    else { if (g.bres) go(margfit_stream_kernel<MOI, RB, 1, true, false>); else go(margfit_stream_kernel<MOI, RB, 1, false, false>); }
  } else {
    if constexpr (RB == 4 || RB == 10) {
      if (q32) { if (g.bres) go(margfit_stream_kernel<MOI, RB, 2, true, true>); else go(margfit_stream_kernel<MOI, RB, 2, false, true>); }
      else { if (g.bres) go(margfit_stream_kernel<MOI, RB, 2, true, false>); else go(margfit_stream_kernel<MOI, RB, 2, false, false>); }
    } else {
      return cudaErrorInvalidValue;   // excluded by fit_stream_supported
    }
  }
  sum_pairs_kernel<<<1, 32, 0, st>>>(part, gx, out2);
  return cudaGetLastError();
}

bool margfit_supported(const DenseView& X, int R) {
  return fit_stream_supported(X, R) && (X.pitch / 4 <= kST || R <= 10);
}

cudaError_t launch_marg_fit_stream(const DenseView& X, int64_t nk, int moi, int S, int qb, const float* lam,
                                   const float* A, const float* B, const float* C, int R, const int32_t* kmap,
                                   int64_t* x1, int64_t* x2, int64_t* x3, double* ws, double* out2,
                                   cudaStream_t st) {
  if (nk <= 0 || !margfit_supported(X, R)) return cudaErrorInvalidValue;
#define SBT_MF(RBV)                                                                                       \
  return moi == 0 ? margfit_rb<RBV, 0>(X, nk, S, qb, lam, A, B, C, R, kmap, x1, x2, x3, ws, out2, st)     \
                  : margfit_rb<RBV, 1>(X, nk, S, qb, lam, A, B, C, R, kmap, x1, x2, x3, ws, out2, st)
  // (an RB = 8 instantiation of the fused kernel crashes ptxas 12.9: R in 5..8 runs at RB = 10)
  // (RB = 8 and 12 instantiations of the two-quad kernel crash ptxas 12.9: R in 5..8 runs at
  // RB = 10, and R = 11, 12 with rows > 2048 floats are not offered: margfit_supported)
  if (R <= 4) { SBT_MF(4); }
  if (R <= 10) { SBT_MF(10); }
  if (R <= 12) { SBT_MF(12); }
  SBT_MF(16);
#undef SBT_MF
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
  int nparts = 0;
  cudaError_t e = fit_pass<RB>(X, lam, A, B, C, R, kmap, ws, &nparts, st);
  if (e != cudaSuccess) return e;
  sum_pairs_kernel<<<1, 32, 0, st>>>(ws, nparts, out2);
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
  if (R <= 10) return fit_partial_rb<10>(X, lam, A, B, C, R, kmap, ws, out2, st);
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
  if (R <= 10) return fit_stream_rb<10>(X, lam, A, B, C, R, ws, relerr, st);
  if (R <= 12) return fit_stream_rb<12>(X, lam, A, B, C, R, ws, relerr, st);
  if (R <= 16) return fit_stream_rb<16>(X, lam, A, B, C, R, ws, relerr, st);
  return cudaErrorInvalidValue;   // callers use the tiled kernel for R > 16
}

}  // namespace sbt
