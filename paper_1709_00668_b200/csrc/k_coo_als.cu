// k_coo_als.cu -- the batched CP-ALS of the r COO summaries (Alg. 1 l.5; R10-R12) as ONE
// persistent cooperative kernel: every iteration and mode of every repetition runs between grid
// barriers instead of ~16 kernel boundaries per iteration (the per-mode pipeline of k_coo.cu's
// piece MTTKRP + k_als_rows.cu's solve steps).  Per mode m:
//
//   A  MTTKRP (coo_piece.cuh): one warp per row piece, grid-stride over the pieces of all
//      repetitions; single-piece rows write M, multi-piece rows their piece partial.
//   -- grid barrier --
//   B  rows: unit = (rep, tile of kTile rows); two threads per row: m = M row (or the row's piece
//      partials summed in piece order), x = m Vi (fp64), X = x; the tile's partial Gram
//      sum_t x_t x_t^T and, for mode 2, the fit inner product sum_t <x_t, m_t> (rows in order).
//   -- grid barrier --
//   C  every block: lambda of every repetition = sqrt(diag of the tile partials summed in tile
//      order); leader block rho (< r): the whole Gram G_m normalised by lambda, for mode 2 the
//      fit and the stop test (|fit - fit_prev| < tol), then Vi of the next mode =
//      (G_o1 * G_o2)^-1 (warp Gauss-Jordan, Jacobi pseudo-inverse fallback R12); other blocks:
//      U_m = fp32(x / lambda) and the padded copy, per (rep, tile).
//   -- grid barrier --
//
// A repetition whose last fit met the stop test is done from the next iteration on (the
// per-mode pipeline's commit step).  Every sum runs in a fixed order: deterministic.  Data
// written inside the kernel is read with ld.cg (L2): L1 is not coherent across SMs.
#include <stdio.h>
#include <stdlib.h>

#include "als_small.cuh"
#include "common.cuh"
#include "coo_piece.cuh"
#include "internal.h"

namespace sbt {

namespace {

constexpr int kPT = 256;   // threads per block
constexpr int kTile = 128; // rows per rows-phase tile (two threads per row)
constexpr int kPairsPerGrab = 8;   // short-piece pairs a warp takes from the MTTKRP work counter

__device__ __forceinline__ void grid_sync(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    // spin on relaxed loads (an acquire load per poll would invalidate this SM's L1 each time,
    // under the feet of the co-resident CTAs still working), then one acquire fence
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    while (v < target) {
      __nanosleep(20);
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

__device__ __forceinline__ int mode_rows(const RowsAls& ra, int m) { return m == 0 ? ra.nI : m == 1 ? ra.nJ : ra.nK; }

// nitems sums over the ntile tile partials at addr(i) + t * stride: two consecutive threads per
// item, thread j summing its half of the tiles in order (loads issued 16 at a time: the sums
// are latency-bound chains of L2 reads), the halves added by one shuffle (a + b on both lanes).
// Used for both the leader's Gram and every block's lambda, so the two agree bit for bit.
template <class Addr, class Out>
__device__ __forceinline__ void tile_sums(int nitems, int ntile, int64_t stride, Addr addr, Out out) {
  const int half = (ntile + 1) / 2;
  const int nrounds = (2 * nitems + blockDim.x - 1) / blockDim.x;
  for (int rd = 0; rd < nrounds; ++rd) {   // uniform trip count: every lane reaches the shuffle
    const int slot = rd * blockDim.x + threadIdx.x;
    const int i = slot >> 1, j = slot & 1;
    double s = 0.0;
    if (i < nitems) {
      const double* p = addr(i);
      const int t1 = min(ntile, (j + 1) * half);
      for (int t0 = j * half; t0 < t1; t0 += 16) {
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = t0 + q < t1 ? __ldcg(p + (int64_t)(t0 + q) * stride) : 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) s += v[q];
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (i < nitems && j == 0) out(i, s);
  }
}

// leader work of repetition rep after the rows phase of mode m: G_m, lambda, fit / stop (m = 2),
// and Vi of mode nm.  sh: >= 8 R^2 + R + 1 doubles of shared memory.
template <int RB>
__device__ void leader_reduce(const RowsAls& ra, int rep, int m, double* sh, bool do_reduce, int nm) {
  const int R = ra.R, npair = R * R;
  double* Gx = sh;                  // [npair + 1]
  double* V = sh + npair + 1;       // [npair]
  double* W = V + npair;            // [2 npair]
  double* Q = W + 2 * npair;        // [npair]
  double* Wg0 = Q + npair;          // [2 npair + R]: Gauss-Jordan [V | I], then its column
  double* Gr = ra.G + (int64_t)rep * 3 * npair;
  if (do_reduce) {
    const int ntile = (mode_rows(ra, m) + kTile - 1) / kTile;
    const double* part = ra.part + (int64_t)rep * ntile * (npair + 1);
    tile_sums(npair + 1, ntile, npair + 1, [&](int i) { return part + i; }, [&](int i, double v) { Gx[i] = v; });
    __syncthreads();
    double* lamL = Wg0;   // [R] lambda
    double* G3 = W;       // [3 npair] the three Grams (W and Q, free until the solve)
    for (int pr = threadIdx.x; pr < npair; pr += blockDim.x) {
      const int f = pr / R, g = pr - f * R;
      double lf = sqrt(Gx[f * R + f]), lg = sqrt(Gx[g * R + g]);
      lf = lf > 0.0 ? lf : 1.0; lg = lg > 0.0 ? lg : 1.0;
      const double gn = Gx[pr] / (lf * lg);
      Gr[m * npair + pr] = gn;
      G3[m * npair + pr] = gn;
    }
    if (threadIdx.x < R) {
      const double l = sqrt(Gx[threadIdx.x * R + threadIdx.x]);
      ra.lam[rep * R + threadIdx.x] = l;
      lamL[threadIdx.x] = l;
    }
    if (m == 2)
      for (int e = threadIdx.x; e < 2 * npair; e += blockDim.x) G3[e] = __ldcg(Gr + e);
    __syncthreads();
    double* terms = V;    // [npair] (free until the solve)
    if (m == 2)
      for (int pr = threadIdx.x; pr < npair; pr += blockDim.x) {
        const int f = pr / R, g = pr - f * R;
        terms[pr] = lamL[f] * lamL[g] * G3[pr] * G3[npair + pr] * G3[2 * npair + pr];
      }
    __syncthreads();
    if (m == 2 && threadIdx.x == 0) {
      // fit = 1 - sqrt(||Y||^2 - 2 <Y, M> + ||M||^2) / ||Y||; <Y, M> = sum x m (lambda cancels),
      // ||M||^2 = lam^T (G0 * G1 * G2) lam, terms summed in (f, g) order
      double mn = 0.0;
      for (int pr = 0; pr < npair; ++pr) mn += terms[pr];
      const double inner = Gx[npair];
      const double y2 = ra.ysq[rep];
      const double res = fmax(0.0, y2 - 2.0 * inner + mn);
      const double fit = y2 > 0.0 ? 1.0 - sqrt(res) / sqrt(y2) : 0.0;
      const int it = ra.iters[rep] + 1;
      ra.iters[rep] = it;
      const double prev = ra.fit[rep];
      ra.fit_prev[rep] = prev;
      ra.fit[rep] = fit;
      bool stop = it >= ra.maxit;
      if (it >= 2 && fabs(fit - prev) < ra.tol) stop = true;
      if (!isfinite(fit)) { ra.flags[rep] |= 2; stop = true; }
      ra.stop[rep] = stop ? 1 : 0;
    }
    __syncthreads();
  }
  // Vi of mode nm = (G_o1 * G_o2)^-1
  const int o1 = nm == 0 ? 1 : 0, o2 = nm == 2 ? 1 : 2;
  for (int e = threadIdx.x; e < npair; e += blockDim.x) V[e] = __ldcg(Gr + o1 * npair + e) * __ldcg(Gr + o2 * npair + e);
  __syncthreads();
  // Gauss-Jordan on [V | I] in shared memory, the register version's arithmetic (row j / pivot,
  // row i -= W_ij row j as an fma): SPD -> every pivot positive, else the pseudo-inverse
  const int Wd = 2 * R;
  double* Wg = Wg0;                   // [R][2R] (W / Q stay free for pinv_R)
  double* fc = Wg + 2 * npair;        // [R]
  __shared__ int s_ok;
  for (int e = threadIdx.x; e < R * Wd; e += blockDim.x) {
    const int i = e / Wd, c = e - i * Wd;
    Wg[e] = c < R ? V[i * R + c] : (c - R == i ? 1.0 : 0.0);
  }
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  for (int j = 0; j < R; ++j) {
    const double piv = Wg[j * Wd + j];
    if (!(piv > 0.0)) { if (threadIdx.x == 0) s_ok = 0; break; }   // uniform: every thread reads piv
    for (int i = threadIdx.x; i < R; i += blockDim.x) fc[i] = Wg[i * Wd + j];
    __syncthreads();
    for (int c = threadIdx.x; c < Wd; c += blockDim.x) Wg[j * Wd + c] = Wg[j * Wd + c] / piv;
    __syncthreads();
    for (int e = threadIdx.x; e < R * Wd; e += blockDim.x) {
      const int i = e / Wd, c = e - i * Wd;
      if (i != j) Wg[e] = fma(-fc[i], Wg[j * Wd + c], Wg[e]);
    }
    __syncthreads();
  }
  __syncthreads();
  double* Vi = ra.Vi + (int64_t)rep * npair;
  if (s_ok) {
    for (int e = threadIdx.x; e < npair; e += blockDim.x) Vi[e] = Wg[(e / R) * Wd + R + (e % R)];
  } else if (threadIdx.x == 0) {
    pinv_R(V, Vi, R, W, Q);
    ra.flags[rep] |= 1;
  }
  __syncthreads();
}

template <int RB>
__global__ void __launch_bounds__(kPT, 3) coo_als_persist_kernel(const __grid_constant__ CooAls ca_p, const __grid_constant__ RowsAls ra_p, unsigned* bar,
                                                                unsigned long long* prof) {
  extern __shared__ __align__(16) double sh[];   // rows phase: xs[kPT][RB + 1]; leader scratch
  __shared__ double s_lam[kMaxReps * RB];
  __shared__ double s_vi[RB * RB];
  __shared__ int64_t s_ps[kTile + 1];   // piece starts of a rows-phase tile
  __shared__ unsigned s_done;
  __shared__ CooAls ca;    // the parameter structs in shared memory: the mode index is dynamic
  __shared__ RowsAls ra;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) { ca = ca_p; ra = ra_p; }
  __syncthreads();
  const int R = ra.R, r = ra.r, npair = R * R;
  unsigned bt = 0;
  // prof (SAMBATEN_COO_ALS_PROFILE): block 0 accumulates the wall time of each phase kind
  unsigned long long tprev = 0;
  auto stamp = [&](int k) {
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (k >= 0) { prof[k] += t - tprev; prof[4 + k] += 1; }
      tprev = t;
    }
  };
  // arrival of every block at the barrier ending phase k: min / max over blocks of (arrival -
  // phase start), summed over phases (prof[8 + k] = sum of the per-phase max, [12 + k] min)
  unsigned long long tstart = 0;
  auto arrive = [&](int k) {
    if (prof) {
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(prof + 16 + k, t - tstart);
        atomicMin(prof + 20 + k, t - tstart);
      }
    }
  };
  // B sub-steps (profiling): max over units of the time from the unit's start to each mark
  unsigned long long tu = 0;
  auto umark = [&](int k) {
    if (prof) {
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (k < 0) tu = t; else atomicMax(prof + 24 + k, t - tu);
      }
    }
  };
  auto phase_start = [&]() {
    if (prof && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tstart));
  };
  auto flush_arrivals = [&](int k) {   // after the barrier: block 0 folds this phase's max/min
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
      prof[8 + k] += atomicExch(prof + 16 + k, 0ull);
      prof[12 + k] += atomicExch(prof + 20 + k, ~0ull);
    }
  };
  auto gsync = [&]() { bt += gridDim.x; grid_sync(bar, bt); };
  stamp(-1);
  if (tid == 0) {
    unsigned dm = 0;
    for (int t = 0; t < r; ++t) dm |= (__ldcg(ra.done + t) != 0 ? 1u : 0u) << t;
    s_done = dm;
  }
  __syncthreads();
  unsigned done = s_done;
  // prologue: Vi of mode 0 from the initial Grams
  if ((int)blockIdx.x < r && !((done >> blockIdx.x) & 1u)) leader_reduce<RB>(ra, blockIdx.x, 0, sh, false, 0);
  gsync();
  stamp(3);
  const unsigned all = r >= 32 ? 0xffffffffu : ((1u << r) - 1u);
  // The leader work of modes 0 and 1 (the mode's Gram and lambda, the next mode's Vi) is only
  // needed by the next mode's rows phase, so the leader blocks do it at the start of the next
  // MTTKRP phase (pending = that mode), hidden behind the other blocks' MTTKRP.  Mode 2's (with
  // the fit and the stop test the next iteration starts from) stays in its own phase C.
  int pending = -1;
  for (int it = 0; it < ra.maxit; ++it) {
    if (it > 0) {   // commit the stop flags of iteration it - 1
      if (tid == 0) {
        unsigned dm = done;
        for (int t = 0; t < r; ++t) dm |= (__ldcg(ra.stop + t) != 0 ? 1u : 0u) << t;
        s_done = dm;
        if (blockIdx.x == 0)
          for (int t = 0; t < r; ++t)
            if ((dm >> t) & 1u) ra.done[t] = 1;
      }
      __syncthreads();
      done = s_done;
    }
    if ((done & all) == all) break;
    for (int m = 0; m < 3; ++m) {
      // ---- A: MTTKRP pieces (leaders first finish the pending mode) ----
      phase_start();
      if (pending >= 0 && (int)blockIdx.x < r && !((done >> blockIdx.x) & 1u))
        leader_reduce<RB>(ra, blockIdx.x, pending, sh, true, m);
      {
        // pieces from work counters (dynamic: Zipf-hot rows make piece costs uneven), the warp
        // pieces first and then the short pieces two at a time (half-warps), so the phase does
        // not end on a long piece taken last
        const CooModePlan& pa = ca.plan[m];
        const int64_t P = __ldcg(pa.pstart + pa.nrow);
        const int64_t nlong = __ldcg(pa.nlist), nshort = __ldcg(pa.nlist + 1);
        unsigned* wq = bar + 1 + 6 * it + 2 * m;
        // warp pieces round-robin (similar costs, random order: no counter traffic), the short
        // pieces from a counter in batches
        const int64_t gw = ((int64_t)blockIdx.x * kPT + tid) >> 5, nw = ((int64_t)gridDim.x * kPT) >> 5;
        for (int64_t q = gw; q < nlong; q += nw) coo_piece_mttkrp<RB>(ca, m, pa.plist[q], lane, done);
        const int64_t nsp = (nshort + 1) / 2;
        for (;;) {
          unsigned q0 = 0;
          if (lane == 0) q0 = atomicAdd(wq + 1, (unsigned)kPairsPerGrab);
          q0 = __shfl_sync(0xffffffffu, q0, 0);
          if ((int64_t)q0 >= nsp) break;
          const int64_t qe = min((int64_t)q0 + kPairsPerGrab, nsp);
          for (int64_t q = q0; q < qe; ++q) {
            const int64_t j = 2 * q + (lane >> 4);
            if (j < nshort) coo_short_half(ca, m, pa.plist[P - 1 - j], lane & 15, done);
          }
        }
      }
      arrive(0);
      gsync();
      stamp(0);
      flush_arrivals(0);
      phase_start();
      // ---- B: rows ----
      const int n = mode_rows(ra, m);
      const int ntile = (n + kTile - 1) / kTile;
      const int units = r * ntile;
      const CooModePlan& pl = ca.plan[m];
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int rep = u / ntile, tile = u - rep * ntile;
        if ((done >> rep) & 1u) continue;
        for (int e = tid; e < npair; e += kPT) s_vi[e] = __ldcg(ra.Vi + (int64_t)rep * npair + e);
        const int row0 = tile * kTile;
        const int nr = min(kTile, n - row0);
        double* ms = sh;                       // [kTile][RB + 1]: m rows
        double* xs = sh + kTile * (RB + 1);    // [kTile][RB + 1]: x rows, then <x, m> in column RB
        // stage the tile's M rows, element-parallel (coalesced; a multi-piece row's piece
        // partials summed in piece order): the rows' piece starts first, then every element's
        // load at once
        umark(-1);
        for (int t = tid; t <= nr; t += kPT) s_ps[t] = __ldg(pl.pstart + (int64_t)rep * n + row0 + t);
        __syncthreads();
        {
          constexpr int kEl = (kTile * RB + kPT - 1) / kPT;
          const double* Mt = ra.M[m] + rep * ra.m_stride[m] + (int64_t)row0 * R;
          double w[kEl];
#pragma unroll
          for (int q = 0; q < kEl; ++q) {
            const int e = tid + q * kPT;
            w[q] = 0.0;
            if (e < nr * R) {
              const int rl = e / R;
              if (s_ps[rl + 1] - s_ps[rl] == 1) w[q] = __ldcg(Mt + e);
            }
          }
#pragma unroll
          for (int q = 0; q < kEl; ++q) {
            const int e = tid + q * kPT;
            if (e < nr * R) {
              const int rl = e / R, f = e - rl * R;
              const int64_t ps = s_ps[rl], np = s_ps[rl + 1] - ps;
              double v = w[q];
              if (np != 1) {
                v = 0.0;   // the piece partials in order, loads eight at a time
                for (int64_t k0 = 0; k0 < np; k0 += 8) {
                  double wp[8];
#pragma unroll
                  for (int k = 0; k < 8; ++k) wp[k] = k0 + k < np ? __ldcg(pl.partial + (ps + k0 + k) * R + f) : 0.0;
#pragma unroll
                  for (int k = 0; k < 8; ++k) v += wp[k];
                }
              }
              ms[rl * (RB + 1) + f] = v;
            }
          }
        }
        __syncthreads();
        umark(0);
        // x = m Vi: two threads per row, each half of the components (g outer: RB / 2
        // independent chains, each in g order)
        {
          constexpr int H = RB / 2 > 0 ? RB / 2 : 1;
          const int rl = tid & (kTile - 1), f0 = (tid / kTile) * H;
          if (rl < nr) {
            const double* mr = ms + rl * (RB + 1);
            double acc[H];
#pragma unroll
            for (int h = 0; h < H; ++h) acc[h] = 0.0;
            for (int g = 0; g < R; ++g) {
              const double mg = mr[g];
#pragma unroll
              for (int h = 0; h < H; ++h)
                if (f0 + h < R) acc[h] += mg * s_vi[g * R + f0 + h];
            }
#pragma unroll
            for (int h = 0; h < H; ++h)
              if (f0 + h < R) xs[rl * (RB + 1) + f0 + h] = acc[h];
          }
        }
        __syncthreads();
        if (tid < nr) {   // <x, m> of the row, components in order
          double xm = 0.0;
          for (int f = 0; f < R; ++f) xm += xs[tid * (RB + 1) + f] * ms[tid * (RB + 1) + f];
          xs[tid * (RB + 1) + RB] = xm;
        }
        double* X = ra.X + (int64_t)rep * ra.x_stride;
#pragma unroll 4
        for (int e = tid; e < nr * R; e += kPT) {   // X rows of the tile, coalesced
          const int rl = e / R, f = e - rl * R;
          X[(int64_t)row0 * R + e] = xs[rl * (RB + 1) + f];
        }
        __syncthreads();
        umark(1);
        double* part = ra.part + ((int64_t)rep * ntile + tile) * (npair + 1);
        for (int pr = tid; pr <= npair; pr += kPT) {
          double s = 0.0;
          if (pr < npair) {   // four interleaved chains (rows t mod 4), combined in a fixed order
            const int f = pr / R, g = pr - f * R;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int t = 0;
            for (; t + 4 <= nr; t += 4) {
              s0 += xs[t * (RB + 1) + f] * xs[t * (RB + 1) + g];
              s1 += xs[(t + 1) * (RB + 1) + f] * xs[(t + 1) * (RB + 1) + g];
              s2 += xs[(t + 2) * (RB + 1) + f] * xs[(t + 2) * (RB + 1) + g];
              s3 += xs[(t + 3) * (RB + 1) + f] * xs[(t + 3) * (RB + 1) + g];
            }
            for (; t < nr; ++t) s0 += xs[t * (RB + 1) + f] * xs[t * (RB + 1) + g];
            s = (s0 + s1) + (s2 + s3);
          } else if (m == 2) {
            for (int t = 0; t < nr; ++t) s += xs[t * (RB + 1) + RB];
          }
          part[pr] = s;
        }
        __syncthreads();
        umark(2);
      }
      arrive(1);
      gsync();
      stamp(1);
      flush_arrivals(1);
      phase_start();
      // ---- C: lambda, leader reduce + next Vi, scale ----
      tile_sums(r * R, ntile, npair + 1,
                [&](int i) { const int rep = i / R, f = i - rep * R;
                             return ra.part + (int64_t)rep * ntile * (npair + 1) + f * R + f; },
                [&](int i, double v) { const int rep = i / R, f = i - rep * R; s_lam[rep * RB + f] = sqrt(v); });
      __syncthreads();
      if (m == 2 && (int)blockIdx.x < r && !((done >> blockIdx.x) & 1u))
        leader_reduce<RB>(ra, blockIdx.x, 2, sh, true, 0);
      {
        const int start = ((int)blockIdx.x - r + (int)gridDim.x * 8) % (int)gridDim.x;
        for (int u = start; u < units; u += gridDim.x) {
          const int rep = u / ntile, tile = u - rep * ntile;
          if ((done >> rep) & 1u) continue;
          const double* X = ra.X + (int64_t)rep * ra.x_stride;
          float* U = ra.U[m] + rep * ra.u_stride[m];
          float* Up = ra.Up[m] + rep * ra.up_stride[m];
          const int row0 = tile * kTile;
          const int nel = (min(row0 + kTile, n) - row0) * R;
#pragma unroll 4
          for (int e = tid; e < nel; e += kPT) {
            const int rl = e / R, f = e - rl * R;
            const int64_t t = (int64_t)row0 * R + e;
            const double l = s_lam[rep * RB + f];
            const double xv = __ldcg(X + t);
            const float uv = __double2float_rn(l > 0.0 ? xv / l : xv);
            U[t] = uv;
            Up[(int64_t)(row0 + rl) * ra.RBp + f] = uv;
          }
        }
      }
      arrive(2);
      gsync();
      stamp(2);
      flush_arrivals(2);
      pending = m < 2 ? m : -1;
    }
  }
}

template <int RB>
size_t persist_smem() { return std::max<size_t>((size_t)2 * kTile * (RB + 1), 8 * RB * RB + RB + 1) * sizeof(double); }

template <int RB>
cudaError_t launch_rb(const CooAls& ca, const RowsAls& ra, unsigned* bar, cudaStream_t st, int* blocks_out,
                      unsigned long long* prof) {
  const size_t smem = persist_smem<RB>();
  cudaError_t e = cudaFuncSetAttribute(coo_als_persist_kernel<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coo_als_persist_kernel<RB>, kPT, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  static const int cap = [] { const char* v = getenv("SAMBATEN_COO_ALS_BPS"); return v ? atoi(v) : 3; }();
  per_sm = std::min(per_sm, std::max(cap, 1));
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = std::max(per_sm * sms, ra.r);
  *blocks_out = blocks;
  e = cudaMemsetAsync(bar, 0, sizeof(unsigned) * coo_als_persist_ctr_words(ra.maxit), st);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kPT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, coo_als_persist_kernel<RB>, ca, ra, bar, prof);
}

}  // namespace

size_t coo_als_persist_ctr_words(int maxit) { return 1 + 6 * (size_t)std::max(maxit, 1); }

size_t coo_als_persist_part_doubles(int maxn, int R, int r) {
  return (size_t)r * ((maxn + kTile - 1) / kTile) * (R * R + 1);
}

bool coo_als_persist_supported(int R) {
  const bool off = getenv("SAMBATEN_COO_ALS_MULTI") != nullptr;   // the per-mode pipeline (read per call)
  return !off && R <= 16;
}

// all iterations of the batched COO ALS in one cooperative launch (R <= 16, padded factors)
cudaError_t launch_coo_als_persist(const CooAls& ca, const RowsAls& ra, unsigned* bar, cudaStream_t st) {
  if (ra.R > 16 || !ra.Up[0] || !ca.Up[0] || ra.r > kMaxReps) return cudaErrorInvalidValue;
  int blocks = 0;
  static unsigned long long* prof = nullptr;
  static const bool want_prof = getenv("SAMBATEN_COO_ALS_PROFILE") != nullptr;
  if (want_prof && !prof && cudaMalloc(&prof, 28 * sizeof(unsigned long long)) != cudaSuccess) prof = nullptr;
  if (prof) {
    cudaMemsetAsync(prof, 0, 20 * sizeof(unsigned long long), st);
    cudaMemsetAsync(prof + 20, 0xff, 4 * sizeof(unsigned long long), st);
    cudaMemsetAsync(prof + 24, 0, 4 * sizeof(unsigned long long), st);
  }
  cudaError_t e;
  switch (ca.RB) {
    case 4: e = launch_rb<4>(ca, ra, bar, st, &blocks, prof); break;
    case 8: e = launch_rb<8>(ca, ra, bar, st, &blocks, prof); break;
    case 12: e = launch_rb<12>(ca, ra, bar, st, &blocks, prof); break;
    case 16: e = launch_rb<16>(ca, ra, bar, st, &blocks, prof); break;
    default: return cudaErrorInvalidValue;
  }
  if (prof && e == cudaSuccess) {
    unsigned long long h[28];
    e = cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    fprintf(stderr, "[coo_als_persist] blocks %d  us: A(mttkrp) %.1f/%llu  B(rows) %.1f/%llu  C(reduce+scale) %.1f/%llu  prologue %.1f\n",
            blocks, h[0] * 1e-3, h[4], h[1] * 1e-3, h[5], h[2] * 1e-3, h[6], h[3] * 1e-3);
    fprintf(stderr, "[coo_als_persist] block arrival (sum over phases) us: A max %.1f min %.1f  B max %.1f min %.1f  C max %.1f min %.1f\n",
            h[8] * 1e-3, h[12] * 1e-3, h[9] * 1e-3, h[13] * 1e-3, h[10] * 1e-3, h[14] * 1e-3);
    fprintf(stderr, "[coo_als_persist] rows unit (max over all units) us: staged %.1f  x %.1f  gram %.1f\n",
            h[24] * 1e-3, h[25] * 1e-3, h[26] * 1e-3);
  }
  return e;
}

}  // namespace sbt
