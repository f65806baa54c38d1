// k_als_cluster.cu -- a4: batched CP-ALS, one thread-block CLUSTER per repetition
// (Alg. 1 l.5 P:213; readings R10-R12).
//
// The r summaries are independent ALS problems ("does not require any
// synchronization").  Each one is owned by a cluster of CS CTAs (CS <= 16) that runs ALL
// iterations in one launch; the CTAs exchange partial results through distributed shared
// memory (DSMEM) and cluster barriers instead of kernel boundaries.
//
// Layouts (written by the gather, k_gather.cu):  Y[u][q][p] (p fastest) and its per-slice
// transpose Yt[u][p][q] (q fastest).  CTA c owns the K' slices u in [u0, u1).  Both
// streaming passes are column-parallel (consecutive threads read consecutive floats of a
// row; no cross-thread reduction inside a row):
//   mode 0 (pass A over Y):   T_u(p,f) = sum_q Y(u,q,p) U1(q,f);  P(p,f) = sum_u U2(u,f) T_u(p,f)
//   mode 1 (pass B over Yt):  D(u,q,f) = sum_p Yt(u,p,q) U0(p,f);  P(q,f) = sum_u U2(u,f) D(u,q,f)
//   mode 2 (no pass):         M2(u,f) = sum_q D(u,q,f) U1(q,f)   (local to the owner of u)
// (U0 is fixed between modes 1 and 2, so D serves both: 2 passes per iteration, not 3.)
// Mode 0/1 step: barrier; CTA c sums the CS partials of its chunk of rows (fixed rank
// order), solves U = M V^-1 (V = Hadamard of the other two Grams, inverted by warp 0 while
// the pass runs; pseudo-inverse fallback R12) and the chunk's partial Gram; barrier; every
// CTA sums the Grams -> lambda (column norms), normalised Gram, and pulls all normalised
// rows into its fp32 copy of U.  Mode 2: solve of the own rows, partial Gram and the fit
// inner product; one barrier.  Every CTA then computes the same fit -> uniform stop test.
// Precision: fp32 products; per-thread fp32 runs of one slice (<= nI or nJ terms), scaled by
// U2 into per-thread fp32 sums over the CTA's <= ceil(K'/CS) slices; fp64 across threads and
// CTAs (fixed order, deterministic); Grams, solves, norms and the fit in fp64.
#include <cooperative_groups.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "als_small.cuh"
#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace sbt {

constexpr int kCT = 512;          // threads per CTA
constexpr int kCW = kCT / 32;     // warps per CTA


constexpr int kTS = 2;            // TMA stages per team
constexpr int kTSA = 2;           // TMA stages of the wide pass A (larger stages, fewer team barriers)

struct ClLayout {
  size_t G, Gp, Gs, Vi, W1, lam, sc, bars, P, Xun, Xun2, Msh, U0s, U1s, U2s, Dsh, stage, total;
  int chunk0, chunk1, ownK, stage_fl, T, NT;
  int NTA, sfla;       // pass A: teams (all warps but the inverse warp), floats per ring stage
  int wideA, RPT, trA; // wide pass A: one team of all warps but the inverse warp, RPT rows per
                       // step (thread = (row offset, column quad)), trA rows per ring stage
};

__host__ __device__ inline size_t al16(size_t b) { return (b + 15) & ~(size_t)15; }
__host__ __device__ inline int imax3(int a, int b, int c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }
__host__ __device__ inline int pitch4(int n) { return (n + 3) & ~3; }

// Teams: warp-aligned groups of T threads, one thread per column quad (4 floats) of the wider
// layout; NT = teams per CTA (<= 15: one named barrier each).
__host__ __device__ inline void cl_teams(int nI, int nJ, int* T, int* NT) {
  const int quads = pitch4(nI > nJ ? nI : nJ) / 4;
  *T = 32 * ((quads + 31) / 32);
  int nt = kCT / *T;
  *NT = nt > 15 ? 15 : nt;
}

// Shared-memory layout; identical on host (sizing) and device.
// nt_cap: at most this many teams (no more than a CTA has slices).
// dsh: D of the own slices (ownK x nJ x RB fp32) in shared memory instead of global.
__host__ __device__ inline ClLayout cl_layout(int nI, int nJ, int nK, int RB, int CS, int stage_fl,
                                              int dsh, int nt_cap = 16) {
  ClLayout L{};
  L.chunk0 = (nI + CS - 1) / CS;
  L.chunk1 = (nJ + CS - 1) / CS;
  L.ownK = (nK + CS - 1) / CS;
  cl_teams(nI, nJ, &L.T, &L.NT);
  if (L.NT > nt_cap) L.NT = nt_cap;
  if (L.NT > L.ownK) L.NT = L.ownK > 0 ? L.ownK : 1;
  const int mrows = imax3(L.chunk0, L.chunk1, L.ownK);
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += al16(b); return r; };
  const size_t RR = (size_t)RB * RB;
  L.G = take(sizeof(double) * 3 * RR);
  L.Gp = take(sizeof(double) * 3 * RR);
  L.Gs = take(sizeof(double) * RR);
  L.Vi = take(sizeof(double) * RR);
  L.W1 = take(sizeof(double) * 2 * RR);       // W1 | W2 (Gauss-Jordan / pinv scratch)
  L.lam = take(sizeof(double) * RB);
  L.sc = take(sizeof(double) * 64);
  L.bars = take(sizeof(unsigned long long) * kTS * 16);
  L.P = take(sizeof(double) * (size_t)(nI > nJ ? nI : nJ) * RB);
  L.Xun = take(sizeof(double) * (size_t)mrows * RB);
  L.Xun2 = take(sizeof(double) * (size_t)L.ownK * RB);
  L.Msh = take(sizeof(double) * (size_t)mrows * RB);
  L.U0s = take(sizeof(float) * (size_t)nI * ((RB + 3) & ~3));
  L.U1s = take(sizeof(float) * (size_t)nJ * ((RB + 3) & ~3));
  L.U2s = take(sizeof(float) * (size_t)L.ownK * RB);
  L.Dsh = take(dsh ? sizeof(float) * (size_t)L.ownK * nJ * RB : 0);
  // per-team TMA rings (kTS stages of whole rows, at least one row of the wider layout); the
  // rings double as the end-of-pass reduction buffer (4 * RB * kCT floats)
  const int rowmax = pitch4(nI > nJ ? nI : nJ);
  L.stage_fl = stage_fl > rowmax ? stage_fl : rowmax;
  const size_t ring = sizeof(float) * (size_t)L.NT * kTS * L.stage_fl;
  const size_t red = sizeof(float) * (size_t)4 * RB * kCT;
  L.stage = take(ring > red ? ring : red);
  L.total = o;
  // pass A: every team of the CTA (all warps but the inverse warp) streams a row range through
  // its own ring of kTS stages carved from the same region (>= one row per stage)
  const size_t region = ring > red ? ring : red;
  L.NTA = (kCW - 1) / (L.T / 32);
  if (L.NTA < 1) L.NTA = 1;
  if (L.NTA > 15) L.NTA = 15;
  L.sfla = (int)(region / (sizeof(float) * kTS * L.NTA)) & ~3;
  if (L.sfla > 12288) L.sfla = 12288;
  if (L.sfla < pitch4(nI)) L.sfla = 0;   // too little room: pass A keeps the slice teams
  // wide pass A: kTSA stages of trA rows (a multiple of RPT when room allows) plus two W
  // buffers of trA rows (W(u,q,:) = U1(q,:) * U2(u,:), row stride wstride(RB))
  {
    const int pA = pitch4(nI), qa = pA / 4;
    L.RPT = (kCT - 32) / qa;
    const size_t regf = region / sizeof(float);
    int tr = (int)(regf / ((size_t)kTSA * pA + 2 * (size_t)((RB + 3) & ~3)));
    if ((size_t)tr * pA * sizeof(float) > (1u << 19)) tr = (int)((1u << 19) / (sizeof(float) * pA));   // mbarrier tx-count
    if (tr >= L.RPT && L.RPT > 0) tr -= tr % L.RPT;
    L.trA = tr;
    L.wideA = L.RPT >= 1 && tr >= 1;
  }
  return L;
}

// ---- mbarrier / TMA bulk-copy helpers (cp.async.bulk, sm_90+) ----------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// rows of RB floats (RB even): 16 B vectors when RB % 4 == 0, else 8 B
template <int RB>
__device__ __forceinline__ void ld_row(const float* p, float (&w)[RB]) {
  if constexpr (RB % 4 == 0) {
#pragma unroll
    for (int f4 = 0; f4 < RB / 4; ++f4) {
      const float4 v = reinterpret_cast<const float4*>(p)[f4];
      w[4 * f4 + 0] = v.x; w[4 * f4 + 1] = v.y; w[4 * f4 + 2] = v.z; w[4 * f4 + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int f2 = 0; f2 < RB / 2; ++f2) {
      const float2 v = reinterpret_cast<const float2*>(p)[f2];
      w[2 * f2 + 0] = v.x; w[2 * f2 + 1] = v.y;
    }
  }
}
// Row stride (floats) of the CTA's U0 / U1 copies and of the wide pass's W rows: RB rounded
// up to a float4 multiple, so a row is whole float4 loads (+ one float2 when RB % 4 == 2).
__host__ __device__ __forceinline__ int wstride(int RB) { return (RB + 3) & ~3; }

template <int RB>
__device__ __forceinline__ void ld_wrow(const float* p, float (&w)[RB]) {
#pragma unroll
  for (int f4 = 0; f4 < RB / 4; ++f4) {
    const float4 v = reinterpret_cast<const float4*>(p)[f4];
    w[4 * f4 + 0] = v.x; w[4 * f4 + 1] = v.y; w[4 * f4 + 2] = v.z; w[4 * f4 + 3] = v.w;
  }
  if constexpr (RB % 4 == 2) {
    const float2 v = reinterpret_cast<const float2*>(p)[RB / 2 - 1];
    w[RB - 2] = v.x; w[RB - 1] = v.y;
  }
}

template <int RB>
__device__ __forceinline__ void st_row(float* p, const float (&w)[RB]) {
  if constexpr (RB % 4 == 0) {
#pragma unroll
    for (int f4 = 0; f4 < RB / 4; ++f4)
      reinterpret_cast<float4*>(p)[f4] = make_float4(w[4 * f4], w[4 * f4 + 1], w[4 * f4 + 2], w[4 * f4 + 3]);
  } else {
#pragma unroll
    for (int f2 = 0; f2 < RB / 2; ++f2) reinterpret_cast<float2*>(p)[f2] = make_float2(w[2 * f2], w[2 * f2 + 1]);
  }
}

// Sum over the cluster's CTAs (fixed rank order) of element idx of an exported smem array;
// the CS remote loads are issued before the ordered additions.
__device__ __noinline__ double cluster_sum(double* local, int idx, int CS) {
  cg::cluster_group cl = cg::this_cluster();
  double v[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) v[c] = c < CS ? cl.map_shared_rank(local, c)[idx] : 0.0;
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 16; ++c)
    if (c < CS) s += v[c];
  return s;
}

// Inverse of the SPD R x R matrix V (R-stride) by Gauss-Jordan without pivoting in one warp
// (every pivot of an SPD matrix is positive; a non-positive pivot means "not positive
// definite" -> pseudo-inverse fallback, R12).  Ag: R x 2R scratch, fc: R doubles.
__device__ __noinline__ bool warp_spd_inverse(const double* V, double* Vi, double* Ag, double* fc,
                                              int R) {
  const int lane = threadIdx.x & 31;
  const int W = 2 * R;
  for (int e = lane; e < R * W; e += 32) {
    const int i = e / W, c = e - i * W;
    Ag[e] = c < R ? V[i * R + c] : (c - R == i ? 1.0 : 0.0);
  }
  __syncwarp();
  bool ok = true;
  for (int j = 0; j < R; ++j) {
    const double piv = Ag[j * W + j];
    if (!(piv > 0.0)) { ok = false; break; }
    for (int i = lane; i < R; i += 32) fc[i] = Ag[i * W + j];
    __syncwarp();
    const double rp = 1.0 / piv;
    for (int c = lane; c < W; c += 32) Ag[j * W + c] *= rp;
    __syncwarp();
    for (int e = lane; e < R * W; e += 32) {
      const int i = e / W, c = e - i * W;
      if (i != j) Ag[e] -= fc[i] * Ag[j * W + c];
    }
    __syncwarp();
  }
  if (ok)
    for (int e = lane; e < R * R; e += 32) {
      const int i = e / R, c = e - i * R;
      Vi[e] = Ag[i * W + R + c];
    }
  __syncwarp();
  return ok;
}

// Register Gauss-Jordan for R <= RB <= 16: lane c < 2R holds column c of [V | I] in
// registers; step j broadcasts the pivot and the R entries of column j by shuffles.
template <int RB>
__device__ __forceinline__ bool warp_spd_inverse_reg(const double* V, double* Vi, int R) {
  const int lane = threadIdx.x & 31;
  double col[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    double v = 0.0;
    if (i < R) v = lane < R ? V[i * R + lane] : (lane - R == i ? 1.0 : 0.0);
    col[i] = v;
  }
  bool ok = true;
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    if (j < R) {
      const double piv = __shfl_sync(0xffffffffu, col[j], j);
      ok = ok && (piv > 0.0);
      double fcol[RB];
#pragma unroll
      for (int i = 0; i < RB; ++i) fcol[i] = __shfl_sync(0xffffffffu, col[i], j);
      col[j] = col[j] * __drcp_rn(piv);   // correctly rounded reciprocal: ~4x shorter chain than a division
#pragma unroll
      for (int i = 0; i < RB; ++i)
        if (i < R && i != j) col[i] = fma(-fcol[i], col[j], col[i]);
    }
  }
  if (ok && lane >= R && lane < 2 * R)
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if (i < R) Vi[i * R + (lane - R)] = col[i];
  __syncwarp();
  return ok;
}

// Warp 0: Vi = (G_o1 * G_o2)^-1 for mode m (Hadamard of the other two normalised Grams).
template <int RB>
__device__ __forceinline__ void warp_normal_inverse(const double* G, int m, int R, double* Vm,
                                                 double* Vi, double* W1, double* fc, int* flags) {
  const int lane = threadIdx.x & 31;
  const int o1 = m == 0 ? 1 : 0, o2 = m == 2 ? 1 : 2;
  for (int idx = lane; idx < R * R; idx += 32) Vm[idx] = G[o1 * RB * RB + idx] * G[o2 * RB * RB + idx];
  __syncwarp();
  bool ok;
  if constexpr (RB <= 16) ok = warp_spd_inverse_reg<RB>(Vm, Vi, R);
  else ok = warp_spd_inverse(Vm, Vi, W1, fc, R);
  if (!ok && lane == 0) {
    pinv_R(Vm, Vi, R, W1, W1 + RB * RB);
    *flags |= 1;
  }
  __syncwarp();
}

#ifdef SBT_ALS_PHASES
__device__ unsigned long long g_als_phase[32];
#define PH(k)                                                                            \
  do {                                                                                   \
    if (tid == 0 && rep == 0 && rank == 0) {                                             \
      const long long t_ = clock64();                                                    \
      atomicAdd(&g_als_phase[k], (unsigned long long)(t_ - ph_t));                       \
      ph_t = t_;                                                                         \
    }                                                                                    \
  } while (0)
#else
#define PH(k) do { } while (0)
#endif

__device__ __forceinline__ void team_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// One streaming pass over the CTA's own slices of a layout Src[u][row][col] (row pitch
// `pitch` floats, multiple of 4, zero padded; slices contiguous).  Team t (T threads, one
// per column quad) owns the slices t, t+NT, ... and streams them through its own kTS-deep
// TMA ring (its thread 0 issues cp.async.bulk copies of whole-row stages; the team syncs
// on a named barrier), so every thread sees whole columns and no reduction inside a slice
// is needed:
//   Pass A (!PASSB): acc(c,f) += Src(u,q,col_c) U1(q,f) U2(u,f)   (Khatri-Rao row formed on
//     the fly), accumulated over the team's slices; P(col,f) = sum over teams (fp64).
//   Pass B (PASSB):  acc(c,f) = sum_p Src(u,p,col_c) U0(p,f) = D(u,col_c,f), stored (fp32,
//     global) at each slice end; P is formed afterwards from D (see mode 1).
// tseq: stages this team has consumed so far (same value in every thread of the team).
template <int RB, bool PASSB>
__device__ __forceinline__ void team_pass(const float* __restrict__ region, int nu, int nrow, int ncol,
                                       int pitch, const float* Uw, const float* U2s, float* rings,
                                       int stage_fl, unsigned long long* bars, int T, int NT,
                                       unsigned tseq, float* Dg, double* P, double* ss = nullptr,
                                       double* s_red = nullptr) {
  const int tid = threadIdx.x;
  // ss (pass B of the first iteration): ||Src||^2 of the CTA's slices on the way -- the four
  // squares of a quad in fp32, widened once per quad; block sum into *ss (fixed order)
  const bool want_ss = PASSB && ss != nullptr;
  double ssd = 0.0;
#ifdef SBT_ALS_PHASES
  const long long tp0 = clock64();
#endif
  const int team = tid / T, lt = tid - team * T;
  const bool in_team = team < NT;
  const bool valid = in_team && 4 * lt < pitch;
  const int trmax = stage_fl / pitch > 0 ? stage_fl / pitch : 1;
  const int nch = (nrow + trmax - 1) / trmax;
  const int tr = (nrow + nch - 1) / nch;
  const int nsl = in_team && team < nu ? (nu - team + NT - 1) / NT : 0;   // slices of this team
  const int total = nsl * nch;
  float* ring = rings + (size_t)(in_team ? team : 0) * kTS * stage_fl;
  unsigned long long* tb = bars + (in_team ? team : 0) * kTS;
  const int bar_id = 1 + team;
  auto issue = [&](int s) {
    const int ul = team + (s / nch) * NT, k = s % nch;
    const int r0 = k * tr, nr = min(tr, nrow - r0);
    const unsigned buf = (tseq + s) % kTS;
    const unsigned bytes = (unsigned)(nr * pitch * sizeof(float));
    mbar_expect_tx(&tb[buf], bytes);
    bulk_g2s(ring + buf * stage_fl, region + ((int64_t)ul * nrow + r0) * pitch, bytes, &tb[buf]);
  };
  if (lt == 0 && total > 0) {
    fence_proxy_async();
    for (int s = 0; s < total && s < kTS; ++s) issue(s);
  }
  float acc[4][RB];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int f = 0; f < RB; ++f) acc[c][f] = 0.f;
  float u2[RB];
  for (int s = 0; s < total; ++s) {
    const int ul = team + (s / nch) * NT, k = s % nch;
    const int r0 = k * tr, nr = min(tr, nrow - r0);
    const unsigned buf = (tseq + s) % kTS;
    if (!PASSB && k == 0) ld_row<RB>(U2s + ul * RB, u2);
#ifdef SBT_ALS_PHASES
    const long long tw0 = clock64();
#endif
    mbar_wait(&tb[buf], ((tseq + s) / kTS) & 1u);
#ifdef SBT_ALS_PHASES
    if (tid == 0 && blockIdx.x == 0) atomicAdd(&g_als_phase[PASSB ? 17 : 16], (unsigned long long)(clock64() - tw0));
#endif
    if (valid) {
      const float* st = ring + buf * stage_fl + 4 * lt;
      const float* wr = Uw + r0 * ((RB + 3) & ~3);
#pragma unroll 2
      for (int row = 0; row < nr; ++row) {
        const float4 y = *reinterpret_cast<const float4*>(st + row * pitch);
        if (want_ss) ssd += (double)fmaf(y.x, y.x, fmaf(y.y, y.y, fmaf(y.z, y.z, y.w * y.w)));
        float w[RB];
        ld_wrow<RB>(wr + row * ((RB + 3) & ~3), w);
        if (!PASSB) {
#pragma unroll
          for (int f = 0; f < RB; ++f) w[f] *= u2[f];
        }
#pragma unroll
        for (int f = 0; f < RB; ++f) {
          acc[0][f] = fmaf(y.x, w[f], acc[0][f]);
          acc[1][f] = fmaf(y.y, w[f], acc[1][f]);
          acc[2][f] = fmaf(y.z, w[f], acc[2][f]);
          acc[3][f] = fmaf(y.w, w[f], acc[3][f]);
        }
      }
    }
    if (PASSB && k == nch - 1 && valid) {   // D(u, col, :) complete
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int col = 4 * lt + c;
        if (col < ncol) {
          st_row<RB>(Dg + ((int64_t)ul * ncol + col) * RB, acc[c]);
        }
#pragma unroll
        for (int f = 0; f < RB; ++f) acc[c][f] = 0.f;
      }
    }
    team_bar(bar_id, T);   // stage consumed by the whole team
    if (lt == 0 && s + kTS < total) {
      fence_proxy_async();
      issue(s + kTS);
    }
  }
#ifdef SBT_ALS_PHASES
  if (tid == 0 && blockIdx.x == 0) atomicAdd(&g_als_phase[PASSB ? 19 : 18], (unsigned long long)(clock64() - tp0));
#endif
  if (want_ss) {
    const double t = block_sum_d(ssd, s_red);
    if (tid == 0) *ss = t;
  }
  if (!PASSB) {
    __syncthreads();   // every team done: rings free (no copy in flight) -> reduction buffer
    float* red = rings;
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int f = 0; f < RB; ++f) red[(c * RB + f) * kCT + tid] = acc[c][f];
    __syncthreads();
    // (c, f) outer, column quad inner: a warp reads consecutive words (conflict-free)
    const int nq = (ncol + 3) >> 2;
    for (int e = tid; e < 4 * RB * nq; e += kCT) {
      const int cf = e / nq, qd = e - cf * nq;
      const int col = 4 * qd + cf / RB, f = cf % RB;
      if (col >= ncol) continue;
      const float* rr = red + cf * kCT + qd;
      double v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = t < NT ? (double)rr[t * T] : 0.0;
      double sum = 0.0;
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (t < NT) sum += v[t];
      P[col * RB + f] = sum;
    }
  }
}

// Pass A with the CTA's row space split into NTA contiguous ranges, one per team (all warps
// but the inverse warp), each streamed through the team's own TMA ring: row g = (u, q) of the
// CTA's own slices (contiguous in Y).  acc(c,f) += Y(u,q,col_c) U1(q,f) U2(u,f);
// P = sum over teams (fp64, fixed order).  Ranges may cross slice boundaries.
__device__ __forceinline__ void pass_a_range(int team, int NTA, int total, int* g0, int* g1) {
  const int L = (total + NTA - 1) / NTA;
  *g0 = min(total, team * L);
  *g1 = min(total, *g0 + L);
}

template <int RB>
__device__ __forceinline__ void team_pass_a(const float* __restrict__ region, int nu, int nrow, int ncol,
                                            int pitch, const float* Uw, const float* U2s, float* rings,
                                            int sfl, unsigned long long* bars, int T, int NTA, unsigned tseq,
                                            double* P) {
  const int tid = threadIdx.x;
  const int team = tid / T, lt = tid - team * T;
  const bool in_team = team < NTA;
  const bool valid = in_team && 4 * lt < pitch;
  const int trmax = sfl / pitch > 0 ? sfl / pitch : 1;
  int g0 = 0, g1 = 0;
  if (in_team) pass_a_range(team, NTA, nu * nrow, &g0, &g1);
  const int total = (g1 - g0 + trmax - 1) / trmax;
  float* ring = rings + (size_t)(in_team ? team : 0) * kTS * sfl;
  unsigned long long* tb = bars + (in_team ? team : 0) * kTS;
  auto issue = [&](int s) {
    const int r0 = g0 + s * trmax, nr = min(trmax, g1 - r0);
    const unsigned buf = (tseq + s) % kTS;
    const unsigned bytes = (unsigned)(nr * pitch * sizeof(float));
    mbar_expect_tx(&tb[buf], bytes);
    bulk_g2s(ring + buf * sfl, region + (int64_t)r0 * pitch, bytes, &tb[buf]);
  };
  if (lt == 0 && total > 0) {
    fence_proxy_async();
    for (int s = 0; s < total && s < kTS; ++s) issue(s);
  }
  float acc[4][RB];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int f = 0; f < RB; ++f) acc[c][f] = 0.f;
  float u2[RB];
  int ul = g0 / nrow, q = g0 - ul * nrow;
  if (in_team && g0 < g1) ld_row<RB>(U2s + ul * RB, u2);
  for (int s = 0; s < total; ++s) {
    const int r0 = g0 + s * trmax, nr = min(trmax, g1 - r0);
    const unsigned buf = (tseq + s) % kTS;
    mbar_wait(&tb[buf], ((tseq + s) / kTS) & 1u);
    if (valid) {
      const float* st = ring + buf * sfl + 4 * lt;
#pragma unroll 2
      for (int row = 0; row < nr; ++row) {
        const float4 y = *reinterpret_cast<const float4*>(st + row * pitch);
        float w[RB];
        ld_wrow<RB>(Uw + q * ((RB + 3) & ~3), w);
#pragma unroll
        for (int f = 0; f < RB; ++f) w[f] *= u2[f];
#pragma unroll
        for (int f = 0; f < RB; ++f) {
          acc[0][f] = fmaf(y.x, w[f], acc[0][f]);
          acc[1][f] = fmaf(y.y, w[f], acc[1][f]);
          acc[2][f] = fmaf(y.z, w[f], acc[2][f]);
          acc[3][f] = fmaf(y.w, w[f], acc[3][f]);
        }
        if (++q == nrow) {   // next slice: its U2 row
          q = 0;
          ++ul;
          if (r0 + row + 1 < g1) ld_row<RB>(U2s + ul * RB, u2);
        }
      }
    } else if (in_team) {
      // lanes without a column still track the slice cursor (uniform control flow)
      q += nr;
      while (q >= nrow) { q -= nrow; ++ul; }
    }
    team_bar(1 + team, T);   // stage consumed by the whole team
    if (lt == 0 && s + kTS < total) {
      fence_proxy_async();
      issue(s + kTS);
    }
  }
  __syncthreads();   // every team done: rings free (no copy in flight) -> reduction buffer
  float* red = rings;
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int f = 0; f < RB; ++f) red[(c * RB + f) * kCT + tid] = acc[c][f];
  __syncthreads();
  // (c, f) outer, column quad inner: a warp reads consecutive words (conflict-free)
  const int nq = (ncol + 3) >> 2;
  for (int e = tid; e < 4 * RB * nq; e += kCT) {
    const int cf = e / nq, qd = e - cf * nq;
    const int col = 4 * qd + cf / RB, f = cf % RB;
    if (col >= ncol) continue;
    const float* rr = red + cf * kCT + qd;
    double v[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = t < NTA ? (double)rr[t * T] : 0.0;
    double sum = 0.0;
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (t < NTA) sum += v[t];
    P[col * RB + f] = sum;
  }
}

// Wide pass A: all warps but the inverse warp form ONE team over the CTA's row space
// (rows g = (u, q) of the own slices, contiguous in Y), streamed through one ring of kTS
// stages of trA rows.  Thread (sr, qd) handles column quad qd of rows sr, sr + RPT, ... of a
// stage, so RPT * quads of the 480 lanes carry columns (>= 94 % for nI >= 100, vs 78 % for a
// warp per row at nI = 100).  W(g, :) = U1(q, :) * U2(u, :) is formed once per row (one thread
// per row, a stage ahead, into the W buffer the previous stage no longer reads) instead of by
// every thread: the inner step is one float4 of Y, the W row and 4 * RB FMAs.
// acc(c, f) += Y(u, q, col_c) W(g, f); P = sum over the RPT row offsets (fp64, fixed order).
template <int RB>
__device__ __forceinline__ void wide_pass_a(const float* __restrict__ region, int nu, int nrow, int pitch,
                                            const float* U1s, const float* U2s, float* rings, int tr,
                                            int RPT, unsigned long long* bars, unsigned seq, double* P,
                                            int ncol) {
  constexpr int TA = kCT - 32;
  constexpr int WS = (RB + 3) & ~3;
  const int tid = threadIdx.x;
  const bool in_team = tid < TA;
  const int quads = pitch / 4;
  const int sr = tid / quads, qd = tid - sr * quads;
  const bool valid = in_team && sr < RPT;
  const int rows = nu * nrow;
  const int nst = (rows + tr - 1) / tr;
  float* W = rings + (size_t)kTSA * tr * pitch;
  const float invn = 1.0f / (float)nrow;
  auto issue = [&](int s) {
    const int r0 = s * tr, nr = min(tr, rows - r0);
    const unsigned buf = (seq + s) % kTSA;
    const unsigned bytes = (unsigned)(nr * pitch * sizeof(float));
    mbar_expect_tx(&bars[buf], bytes);
    bulk_g2s(rings + (size_t)buf * tr * pitch, region + (int64_t)r0 * pitch, bytes, &bars[buf]);
  };
  auto make_w = [&](int s) {   // one thread per row of stage s
    const int r0 = s * tr, nr = min(tr, rows - r0);
    float* w = W + (size_t)(s & 1) * tr * WS;
    for (int row = tid; row < nr; row += TA) {
      const int g = r0 + row;
      int ul = __float2int_rz((float)g * invn);
      if (ul * nrow > g) --ul;
      else if ((ul + 1) * nrow <= g) ++ul;
      const int q = g - ul * nrow;
      float a[RB], b[RB];
      ld_wrow<RB>(U1s + q * WS, a);
      ld_row<RB>(U2s + ul * RB, b);
#pragma unroll
      for (int f = 0; f < RB; ++f) a[f] *= b[f];
      float* wr = w + row * WS;
#pragma unroll
      for (int f4 = 0; f4 < RB / 4; ++f4)
        reinterpret_cast<float4*>(wr)[f4] = make_float4(a[4 * f4], a[4 * f4 + 1], a[4 * f4 + 2], a[4 * f4 + 3]);
      if constexpr (RB % 4 == 2) reinterpret_cast<float2*>(wr)[RB / 2 - 1] = make_float2(a[RB - 2], a[RB - 1]);
    }
  };
  float acc[4][RB];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int f = 0; f < RB; ++f) acc[c][f] = 0.f;
  if (in_team) {
    if (tid == 0 && nst > 0) {
      fence_proxy_async();
      for (int s = 0; s < nst && s < kTSA; ++s) issue(s);
    }
#ifdef SBT_ALS_PHASES
    const long long tp0 = clock64();
    long long tw = 0, tb = 0;
#endif
    if (nst > 0) make_w(0);
    team_bar(1, TA);   // W of stage 0
    for (int s = 0; s < nst; ++s) {
      const int nr = min(tr, rows - s * tr);
      const unsigned buf = (seq + s) % kTSA;
      if (s + 1 < nst) make_w(s + 1);   // its W buffer was last read in stage s - 1
#ifdef SBT_ALS_PHASES
      const long long tw0 = clock64();
#endif
      mbar_wait(&bars[buf], ((seq + s) / kTSA) & 1u);
#ifdef SBT_ALS_PHASES
      tw += clock64() - tw0;
#endif
      if (valid) {
        const float* st = rings + (size_t)buf * tr * pitch + 4 * qd;
        const float* w = W + (size_t)(s & 1) * tr * WS;
#pragma unroll 2
        for (int row = sr; row < nr; row += RPT) {
          const float4 y = *reinterpret_cast<const float4*>(st + row * pitch);
          float wv[RB];
          ld_wrow<RB>(w + row * WS, wv);
#pragma unroll
          for (int f = 0; f < RB; ++f) {
            acc[0][f] = fmaf(y.x, wv[f], acc[0][f]);
            acc[1][f] = fmaf(y.y, wv[f], acc[1][f]);
            acc[2][f] = fmaf(y.z, wv[f], acc[2][f]);
            acc[3][f] = fmaf(y.w, wv[f], acc[3][f]);
          }
        }
      }
#ifdef SBT_ALS_PHASES
      const long long tb0 = clock64();
#endif
      team_bar(1, TA);   // stage s consumed, W of stage s + 1 complete
#ifdef SBT_ALS_PHASES
      tb += clock64() - tb0;
#endif
      if (tid == 0 && s + kTSA < nst) {
        fence_proxy_async();
        issue(s + kTSA);
      }
    }
#ifdef SBT_ALS_PHASES
    if ((tid == 0 || tid == 448) && blockIdx.x == 0) {
      atomicAdd(&g_als_phase[tid == 0 ? 16 : 23], (unsigned long long)tw);
      atomicAdd(&g_als_phase[tid == 0 ? 18 : 24], (unsigned long long)(clock64() - tp0));
      atomicAdd(&g_als_phase[tid == 0 ? 25 : 26], (unsigned long long)tb);
    }
#endif
  }
  __syncthreads();   // no copy in flight: the ring region becomes the reduction buffer
  float* red = rings;
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int f = 0; f < RB; ++f) red[(c * RB + f) * kCT + tid] = acc[c][f];
  __syncthreads();
  // (c, f) outer, column quad inner: a warp reads consecutive words (conflict-free)
  const int nq = (ncol + 3) >> 2;
  for (int e = tid; e < 4 * RB * nq; e += kCT) {
    const int cf = e / nq, qd = e - cf * nq;
    const int col = 4 * qd + cf / RB, f = cf % RB;
    if (col >= ncol) continue;
    const float* rr = red + cf * kCT + qd;
    double sum = 0.0;
    for (int t = 0; t < RPT; ++t) sum += (double)rr[t * quads];
    P[col * RB + f] = sum;
  }
}

__device__ __forceinline__ int team_stages_a(int team, int NTA, int total, int pitch, int sfl) {
  const int trmax = sfl / pitch > 0 ? sfl / pitch : 1;
  int g0, g1;
  pass_a_range(team, NTA, total, &g0, &g1);
  return (g1 - g0 + trmax - 1) / trmax;
}

// stages a team consumes in one pass (the same formula as in team_pass)
__device__ __forceinline__ int team_stages(int team, int nu, int NT, int nrow, int pitch, int stage_fl) {
  const int trmax = stage_fl / pitch > 0 ? stage_fl / pitch : 1;
  const int nch = (nrow + trmax - 1) / trmax;
  const int nsl = team < nu ? (nu - team + NT - 1) / NT : 0;
  return nsl * nch;
}

// Grid communication (GRID = true): the CS CTAs of a repetition are ordinary CTAs of one
// co-resident (cooperative) grid instead of a thread-block cluster, so a repetition can span
// more SMs than a cluster slot allows (148 / r of them).  What the cluster path reads from its
// peers' shared memory (partial MTTKRPs P, partial Grams Gp, scalars sc) each CTA also exports
// to its slot of a global buffer; solved rows are pushed to a global copy of U_m; the cluster
// barrier becomes a per-repetition arrival counter (release / acquire at gpu scope).  Peer
// data is read with ld.global.cg (L2; L1 is not coherent across SMs).
struct GridComm {
  double* x;          // [r][CS][xstride] exported P | Gp | sc
  float* u;           // [r][2][max(nI, nJ) * US] pushed rows of U_0, U_1
  unsigned* bar;      // [r] arrival counters (zeroed before the launch)
  int xstride;        // doubles per CTA slot
  int offP, offG, offS;
  int ustride;        // floats per (rep, mode) row block
};

__device__ __forceinline__ void grid_rep_sync(unsigned* ctr, unsigned target) {
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

template <int RB, bool GRID>
__global__ void __launch_bounds__(kCT, 1) als_cluster_kernel(DenseAls a, int CS, float* Dglob,
                                                             int stage_fl, int dshw, GridComm gc) {
  // dshw: bit 0 = D in shared memory (plan), bit 1 = narrow pass A (SAMBATEN_ALS_NARROW_A)
  const int dsh = dshw & 1;
  const int rank = GRID ? (int)(blockIdx.x % CS) : (int)cg::this_cluster().block_rank();
  unsigned bar_target = 0;
  auto csync = [&]() {
    if constexpr (GRID) {
      bar_target += (unsigned)CS;
      grid_rep_sync(gc.bar + blockIdx.x / CS, bar_target);
    } else {
      cg::this_cluster().sync();
    }
  };
  double* gx_me = GRID ? gc.x + ((int64_t)(blockIdx.x / CS) * CS + rank) * gc.xstride : nullptr;
  double* gx_rep = GRID ? gc.x + (int64_t)(blockIdx.x / CS) * CS * gc.xstride : nullptr;
  // sum over the repetition's CTAs (fixed rank order) of element idx of an exported array
  auto csum = [&](double* local, int goff, int idx) -> double {
    if constexpr (GRID) {
      double v[16];
      double s = 0.0;
      int c = 0;
      for (; c + 16 <= CS; c += 16) {
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = __ldcg(gx_rep + (int64_t)(c + t) * gc.xstride + goff + idx);
#pragma unroll
        for (int t = 0; t < 16; ++t) s += v[t];
      }
      for (; c < CS; ++c) s += __ldcg(gx_rep + (int64_t)c * gc.xstride + goff + idx);
      return s;
    } else {
      (void)goff;
      return cluster_sum(local, idx, CS);
    }
  };
  const int rep = blockIdx.x / CS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = a.R, nI = a.nI, nJ = a.nJ, nK = a.nK;
  const ClLayout Ly = cl_layout(nI, nJ, nK, RB, CS, stage_fl, dsh);
  extern __shared__ __align__(16) unsigned char smem[];
  double* G = reinterpret_cast<double*>(smem + Ly.G);        // [3][RB*RB] normalised Grams (R-stride)
  double* Gp = reinterpret_cast<double*>(smem + Ly.Gp);      // [3][RB*RB] partial Grams (exported)
  double* Gs = reinterpret_cast<double*>(smem + Ly.Gs);
  double* Vi = reinterpret_cast<double*>(smem + Ly.Vi);
  double* W1 = reinterpret_cast<double*>(smem + Ly.W1);
  double* lam = reinterpret_cast<double*>(smem + Ly.lam);
  double* sc = reinterpret_cast<double*>(smem + Ly.sc);      // [0] ysq, [1] inner (exported)
  double* P = reinterpret_cast<double*>(smem + Ly.P);        // partial MTTKRP (exported)
  double* Xun = reinterpret_cast<double*>(smem + Ly.Xun);    // solved chunk rows (exported)
  double* Xun2 = reinterpret_cast<double*>(smem + Ly.Xun2);  // solved mode-2 rows (local)
  double* Msh = reinterpret_cast<double*>(smem + Ly.Msh);
  float* U0s = reinterpret_cast<float*>(smem + Ly.U0s);
  float* U1s = reinterpret_cast<float*>(smem + Ly.U1s);
  float* U2s = reinterpret_cast<float*>(smem + Ly.U2s);
  float* ring = reinterpret_cast<float*>(smem + Ly.stage);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + Ly.bars);
  __shared__ double s_fc[kMaxR];
  __shared__ double s_linv[kMaxR];   // 1 / lambda_f (1 for a zero column)
  __shared__ double s_red[32];
  __shared__ int s_flags, s_stop;
  __shared__ double s_fit, s_inner;
#ifdef SBT_ALS_PHASES
  long long ph_t = clock64();
#endif

  const float* Y = a.Y + (int64_t)rep * a.y_stride;
  const float* Yt = a.Yt + (int64_t)rep * a.y_stride;
  const int u0 = min(nK, rank * Ly.ownK), u1 = min(nK, u0 + Ly.ownK);
  const int nu = u1 - u0;
  const int pI = pitch4(nI), pJ = pitch4(nJ);
  // own regions of the two layouts (16 B aligned: pitches and y_stride are multiples of 4)
  const float* regA = Y + (int64_t)u0 * nJ * pI;
  const float* regB = Yt + (int64_t)u0 * nI * pJ;
  // D of the own slices: shared memory when it fits (plan), else global (L2-resident)
  float* D = dsh ? reinterpret_cast<float*>(smem + Ly.Dsh) : Dglob + ((int64_t)rep * nK + u0) * nJ * RB;
  const int myteam = tid / Ly.T;
  unsigned tseq = 0;                                       // TMA stages this team consumed
  unsigned seqA = 0;                                       // stages of the wide pass A (barrier set 15)
  const bool wideA = Ly.wideA && !(dshw & 2);
  float* gU0 = a.U[0] + rep * a.u_stride[0];
  float* gU1 = a.U[1] + rep * a.u_stride[1];
  float* gU2 = a.U[2] + rep * a.u_stride[2];
  const int RR = R * R;
  constexpr int US = (RB + 3) & ~3;   // row stride of U0s / U1s

  // ---- initial factors (zero-padded to RB columns), Grams, ||Y||^2 -------------------------
  for (int e = tid; e < nI * US; e += kCT) {
    const int p = e / US, f = e - p * US;
    U0s[e] = f < R ? gU0[(int64_t)p * R + f] : 0.f;
  }
  for (int e = tid; e < nJ * US; e += kCT) {
    const int q = e / US, f = e - q * US;
    U1s[e] = f < R ? gU1[(int64_t)q * R + f] : 0.f;
  }
  for (int e = tid; e < nu * RB; e += kCT) {
    const int ul = e / RB, f = e - ul * RB;
    U2s[e] = f < R ? gU2[(int64_t)(u0 + ul) * R + f] : 0.f;
  }
  if (tid == 0) {
    s_flags = 0; s_stop = 0;
    for (int b = 0; b < kTS * 16; ++b) mbar_init(&bars[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
#pragma unroll 1
  for (int pr = tid; pr < 3 * RR; pr += kCT) {
    const int m = pr / RR, fg = pr - m * RR, f = fg / R, g = fg - f * R;
    double s = 0.0;
    if (m == 0) for (int p = 0; p < nI; ++p) s += (double)U0s[p * US + f] * (double)U0s[p * US + g];
    if (m == 1) for (int q = 0; q < nJ; ++q) s += (double)U1s[q * US + f] * (double)U1s[q * US + g];
    if (m == 2) for (int u = 0; u < nK; ++u) s += (double)gU2[(int64_t)u * R + f] * (double)gU2[(int64_t)u * R + g];
    G[m * RB * RB + fg] = s;
  }
  csync();
  double ysq = 0.0;   // ||Y||^2: formed in the first iteration's pass B (mode 1)
  PH(0);

  double fit = 0.0, fit_prev = 0.0;
  int it = 0;
#pragma unroll 1
  for (;;) {
    // ================================ mode 0 and mode 1 ================================
#pragma unroll 1
    for (int m = 0; m < 2; ++m) {
      const int n = m == 0 ? nI : nJ;
      const int ch = m == 0 ? Ly.chunk0 : Ly.chunk1;
      // warp 0: Vi = (G_o1 * G_o2)^-1 while the other warps stream
#ifdef SBT_ALS_PHASES
      const long long ti0 = clock64();
#endif
      if (warp == kCW - 1) warp_normal_inverse<RB>(G, m, R, Gs, Vi, W1, s_fc, &s_flags);
#ifdef SBT_ALS_PHASES
      if (warp == kCW - 1 && lane == 0 && rep == 0 && rank == 0)
        atomicAdd(&g_als_phase[27 + m], (unsigned long long)(clock64() - ti0));
#endif
      if (m == 0) {
        if (wideA) {
          wide_pass_a<RB>(regA, nu, nJ, pI, U1s, U2s, ring, Ly.trA, Ly.RPT, bars + 15 * kTS, seqA, P, nI);
          seqA += (unsigned)((nu * nJ + Ly.trA - 1) / Ly.trA);
        } else if (Ly.sfla > 0) {
          team_pass_a<RB>(regA, nu, nJ, nI, pI, U1s, U2s, ring, Ly.sfla, bars, Ly.T, Ly.NTA, tseq, P);
          if (myteam < Ly.NTA) tseq += team_stages_a(myteam, Ly.NTA, nu * nJ, pI, Ly.sfla);
        } else {
          team_pass<RB, false>(regA, nu, nJ, nI, pI, U1s, U2s, ring, Ly.stage_fl, bars, Ly.T, Ly.NT,
                               tseq, D, P);
          if (myteam < Ly.NT) tseq += team_stages(myteam, nu, Ly.NT, nJ, pI, Ly.stage_fl);
        }
        __syncthreads();   // the rings (reduction buffer) are re-armed by the next pass
        PH(1);
      } else {
        team_pass<RB, true>(regB, nu, nI, nJ, pJ, U0s, U2s, ring, Ly.stage_fl, bars, Ly.T, Ly.NT,
                            tseq, D, P, it == 0 ? sc : nullptr, s_red);
        if (it == 0 && tid == 0 && GRID) gx_me[gc.offS + 0] = sc[0];
        if (myteam < Ly.NT) tseq += team_stages(myteam, nu, Ly.NT, nI, pJ, Ly.stage_fl);
        __syncthreads();   // D of the own slices complete (global, visible to the CTA)
        // P(q,f) = sum_{own u} U2(u,f) D(u,q,f)   (fixed order; an fp32 run of <= ceil(K'/CS)
        // terms, like the passes' per-thread runs, widened once)
        for (int e = tid; e < nJ * RB; e += kCT) {
          const int f = e % RB;
          float s = 0.f;
          for (int ul = 0; ul < nu; ++ul) s = fmaf(U2s[ul * RB + f], D[(int64_t)ul * nJ * RB + e], s);
          P[e] = (double)s;
        }
        PH(6);
      }
      if constexpr (GRID) {   // export the partial MTTKRP
        const int np = (m == 0 ? nI : nJ) * RB;
        for (int e = tid; e < np; e += kCT) gx_me[gc.offP + e] = P[e];
      }
      csync();   // S1: partials of every CTA complete
      if (m == 1 && it == 0) ysq = csum(sc, gc.offS, 0);
      PH(m == 0 ? 2 : 8);
      // ---- rows [c0, c1) of this mode: sum the CS partials, solve, partial Gram ----
      const int c0 = min(n, rank * ch), c1 = min(n, c0 + ch);
      const int nr = c1 - c0;
#pragma unroll 1
      for (int e = tid; e < nr * R; e += kCT) {
        const int pl = e / R, f = e - pl * R;
        Msh[pl * RB + f] = csum(P, gc.offP, (c0 + pl) * RB + f);
      }
      __syncthreads();
      float* Us = m == 0 ? U0s : U1s;
#pragma unroll 1
      for (int e = tid; e < nr * R; e += kCT) {
        const int pl = e / R, f = e - pl * R;
        double s = 0.0;
        for (int g = 0; g < R; ++g) s += Msh[pl * RB + g] * Vi[g * R + f];
        Xun[pl * RB + f] = s;
        // push the solved row (unnormalised, fp32) into every CTA's copy of U_m: no CTA reads
        // U_m between S1 and S2 (pass A reads U1/U2, pass B U0/U2), and S2 publishes the stores
        const float xf = __double2float_rn(s);
        if constexpr (GRID) {
          gc.u[((int64_t)(blockIdx.x / CS) * 2 + m) * gc.ustride + (c0 + pl) * US + f] = xf;
        } else {
          cg::cluster_group cluster = cg::this_cluster();
          for (int c = 0; c < CS; ++c) cluster.map_shared_rank(Us, c)[(c0 + pl) * US + f] = xf;
        }
      }
      __syncthreads();
#pragma unroll 1
      for (int pr = tid; pr < RR; pr += kCT) {
        const int f = pr / R, g = pr - f * R;
        double s = 0.0;
        for (int pl = 0; pl < nr; ++pl) s += Xun[pl * RB + f] * Xun[pl * RB + g];
        Gp[m * RB * RB + pr] = s;
        if (GRID) gx_me[gc.offG + m * RB * RB + pr] = s;
      }
      PH(m == 0 ? 3 : 9);
      csync();   // S2: solved rows and partial Grams of every CTA complete
      PH(m == 0 ? 4 : 10);
      if constexpr (GRID) {   // pull every CTA's solved rows into the local copy of U_m
        const float* src = gc.u + ((int64_t)(blockIdx.x / CS) * 2 + m) * gc.ustride;
        for (int e = tid; e < n * US; e += kCT) {
          const int p = e / US, f = e - p * US;
          if (f < R) Us[e] = __ldcg(src + e);
        }
      }
#pragma unroll 1
      for (int pr = tid; pr < RR; pr += kCT) Gs[pr] = csum(Gp, gc.offG, m * RB * RB + pr);
      __syncthreads();
      if (tid < R) {
        lam[tid] = sqrt(Gs[tid * R + tid]);
        s_linv[tid] = lam[tid] > 0.0 ? __drcp_rn(lam[tid]) : 1.0;
      }
      __syncthreads();
#pragma unroll 1
      for (int pr = tid; pr < RR; pr += kCT) {
        const int f = pr / R, g = pr - f * R;
        G[m * RB * RB + pr] = Gs[pr] * (s_linv[f] * s_linv[g]);
      }
      if (m == 1) __syncthreads();   // G_1 complete: warp 15 inverts V_2 = G_0 * G_1 below
      if (m == 0) {
#pragma unroll 1
        for (int e = tid; e < n * R; e += kCT) {
          const int p = e / R, f = e - p * R;
          Us[p * US + f] = __double2float_rn((double)Us[p * US + f] * s_linv[f]);
        }
      } else if (warp < kCW - 1) {
        // the 12 warps off the inverting warp's scheduler (warp % 4 != 3) normalise U_1: the
        // inverse is a latency chain and gets its sub-partition's issue slots to itself
        if ((warp & 3) != 3) {
          const int wt = warp - (warp >> 2);   // 0..11
#pragma unroll 1
          for (int e = wt * 32 + lane; e < n * R; e += 12 * 32) {
            const int p = e / R, f = e - p * R;
            Us[p * US + f] = __double2float_rn((double)Us[p * US + f] * s_linv[f]);
          }
        }
      } else {
        // V_2 = (G_0 * G_1)^-1 overlaps the normalisation of U_1 and the M2 loop below
#ifdef SBT_ALS_PHASES
        const long long tinv0 = clock64();
#endif
        warp_normal_inverse<RB>(G, 2, R, Gs, Vi, W1, s_fc, &s_flags);
#ifdef SBT_ALS_PHASES
        if (lane == 0 && rep == 0 && rank == 0) atomicAdd(&g_als_phase[20], (unsigned long long)(clock64() - tinv0));
#endif
      }
      if (m == 0) __syncthreads();
      else if (warp < kCW - 1) team_bar(1, kCT - 32);   // U_1 normalised (the inverting warp runs on)
      PH(m == 0 ? 5 : 11);
    }
    // ==================================== mode 2 ====================================
#ifdef SBT_ALS_PHASES
    const long long tinv0 = clock64();
    if (tid == 0 && rep == 0 && rank == 0) atomicAdd(&g_als_phase[22], 1ull);
#endif
    // M2(u,f) = sum_q D(u,q,f) U1(q,f) for the own slices: a warp per slice (the 12 warps
    // off the scheduler of warp 15, which is still inverting V2): lane partials over
    // q = lane + 32 t in fp32 (<= nJ / 32 terms), then one fp64 butterfly per f
#pragma unroll 1
    for (int ul = warp - (warp >> 2); (warp & 3) != 3 && ul < nu; ul += 12) {   // the 12 warps off the inverse's scheduler
      const float* d = D + (int64_t)ul * nJ * RB;
      float pa[RB];
#pragma unroll
      for (int f = 0; f < RB; ++f) pa[f] = 0.f;
      for (int q = lane; q < nJ; q += 32) {
        float dv[RB], uv[RB];
        ld_row<RB>(d + (int64_t)q * RB, dv);
        ld_wrow<RB>(U1s + q * US, uv);
#pragma unroll
        for (int f = 0; f < RB; ++f) pa[f] = fmaf(dv[f], uv[f], pa[f]);
      }
      double sv[RB];
#pragma unroll
      for (int f = 0; f < RB; ++f) sv[f] = (double)pa[f];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int f = 0; f < RB; ++f) sv[f] += __shfl_xor_sync(0xffffffffu, sv[f], o);
      if (lane == 0)
#pragma unroll
        for (int f = 0; f < RB; ++f) Msh[ul * RB + f] = sv[f];
    }
#ifdef SBT_ALS_PHASES
    if (tid == 0 && rep == 0 && rank == 0) atomicAdd(&g_als_phase[21], (unsigned long long)(clock64() - tinv0));
#endif
    __syncthreads();
    PH(12);
#pragma unroll 1
    for (int e = tid; e < nu * R; e += kCT) {
      const int ul = e / R, f = e - ul * R;
      double s = 0.0;
      for (int g = 0; g < R; ++g) s += Msh[ul * RB + g] * Vi[g * R + f];
      Xun2[ul * RB + f] = s;
    }
    __syncthreads();
    {
      double inner = 0.0;
      for (int e = tid; e < nu * R; e += kCT) {
        const int ul = e / R, f = e - ul * R;
        inner += Xun2[ul * RB + f] * Msh[ul * RB + f];
      }
      inner = block_sum_d(inner, s_red);
      if (tid == 0) { sc[1] = inner; if (GRID) gx_me[gc.offS + 1] = inner; }
    }
#pragma unroll 1
    for (int pr = tid; pr < RR; pr += kCT) {
      const int f = pr / R, g = pr - f * R;
      double s = 0.0;
      for (int ul = 0; ul < nu; ++ul) s += Xun2[ul * RB + f] * Xun2[ul * RB + g];
      Gp[2 * RB * RB + pr] = s;
      if (GRID) gx_me[gc.offG + 2 * RB * RB + pr] = s;
    }
    PH(13);
    csync();   // S3
    PH(14);
#pragma unroll 1
    for (int pr = tid; pr < RR; pr += kCT) Gs[pr] = csum(Gp, gc.offG, 2 * RB * RB + pr);
    if (tid == kCT - 1) s_inner = csum(sc, gc.offS, 1);   // the fit's <Y, M>, fetched alongside
    __syncthreads();
    if (tid < R) {
      lam[tid] = sqrt(Gs[tid * R + tid]);
      s_linv[tid] = lam[tid] > 0.0 ? __drcp_rn(lam[tid]) : 1.0;
    }
    __syncthreads();
    if (warp < kCW - 1) {
#pragma unroll 1
      for (int pr = tid; pr < RR; pr += kCT - 32) {
        const int f = pr / R, g = pr - f * R;
        G[2 * RB * RB + pr] = Gs[pr] * (s_linv[f] * s_linv[g]);
      }
#pragma unroll 1
      for (int e = tid; e < nu * R; e += kCT - 32) {
        const int ul = e / R, f = e - ul * R;
        U2s[ul * RB + f] = __double2float_rn(Xun2[ul * RB + f] * s_linv[f]);
      }
    } else {
      // fit (the last warp, overlapping the two loops above; every CTA computes the same
      // value -> uniform control flow).  G_2 formed here as the loop above forms it.
      double mn = 0.0;
      for (int pr = lane; pr < RR; pr += 32) {
        const int f = pr / R, g = pr - f * R;
        const double g2 = Gs[pr] * (s_linv[f] * s_linv[g]);
        mn += lam[f] * lam[g] * G[pr] * G[RB * RB + pr] * g2;
      }
      mn = warp_sum_d(mn);
      const double inner = s_inner;
      if (lane == 0) {
        const double res = fmax(0.0, ysq - 2.0 * inner + mn);
        const double f = ysq > 0.0 ? 1.0 - sqrt(res) / sqrt(ysq) : 0.0;
        s_fit = f;
        const int itn = it + 1;
        int stop = itn >= a.maxit;
        if (itn >= 2 && fabs(f - fit) < a.tol) stop = 1;
        if (!isfinite(f)) { stop = 1; s_flags |= 2; }
        s_stop = stop;
      }
    }
    __syncthreads();
    fit_prev = fit;
    fit = s_fit;
    ++it;
    PH(15);
    if (s_stop) break;
  }
  // ---- write back: U0 / U1 chunks, own U2 rows, lambda, fit, iterations -------------------
  {
    const int c0 = min(nI, rank * Ly.chunk0), c1 = min(nI, c0 + Ly.chunk0);
    for (int e = tid; e < (c1 - c0) * R; e += kCT) {
      const int pl = e / R, f = e - pl * R;
      gU0[(int64_t)(c0 + pl) * R + f] = U0s[(c0 + pl) * US + f];
    }
    const int d0 = min(nJ, rank * Ly.chunk1), d1 = min(nJ, d0 + Ly.chunk1);
    for (int e = tid; e < (d1 - d0) * R; e += kCT) {
      const int ql = e / R, f = e - ql * R;
      gU1[(int64_t)(d0 + ql) * R + f] = U1s[(d0 + ql) * US + f];
    }
    for (int e = tid; e < nu * R; e += kCT) {
      const int ul = e / R, f = e - ul * R;
      gU2[(int64_t)(u0 + ul) * R + f] = U2s[ul * RB + f];
    }
  }
  if (rank == 0) {
    if (tid < R) a.lam[rep * R + tid] = lam[tid];
    for (int pr = tid; pr < 3 * RR; pr += kCT) {
      const int m = pr / RR, fg = pr - m * RR;
      a.G[(int64_t)rep * 3 * RR + pr] = G[m * RB * RB + fg];
    }
    if (tid == 0) {
      a.fit[rep] = fit; a.fit_prev[rep] = fit_prev; a.iters[rep] = it; a.flags[rep] = s_flags;
      a.ysq[rep] = ysq; a.done[rep] = 1;
    }
  }
  if constexpr (!GRID) cg::this_cluster().sync();   // keep every CTA's shared memory alive until all remote reads are done
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
constexpr size_t kSmemCap = 227 * 1024 - 1024;   // minus the kernel's static smem

static int rb_of(int R) {
  return R <= 4 ? 4 : R <= 8 ? 8 : R <= 10 ? 10 : R <= 12 ? 12 : R <= 16 ? 16 : R <= 24 ? 24 : 32;
}

template <int RB, bool GRID>
static cudaError_t cluster_setup(int CS, size_t smem) {
  auto k = als_cluster_kernel<RB, GRID>;
  (void)smem;   // always allow the cap: plans of several shapes share the kernel
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap);
  if (e != cudaSuccess) return e;
  if (!GRID && CS > 8) e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}

// cluster launch (one cluster of CS CTAs per repetition) or grid launch (cooperative: every CTA
// co-resident, CS consecutive CTAs per repetition)
static void fill_cfg(cudaLaunchConfig_t* cfg, cudaLaunchAttribute* attr, int CS, int nclusters,
                     size_t smem, cudaStream_t st, bool grid = false) {
  *cfg = cudaLaunchConfig_t{};
  cfg->gridDim = dim3((unsigned)(CS * nclusters), 1, 1);
  cfg->blockDim = dim3(kCT, 1, 1);
  cfg->dynamicSmemBytes = smem;
  cfg->stream = st;
  if (grid) {
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
  } else {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
  }
  cfg->attrs = attr;
  cfg->numAttrs = 1;
}

// shared-memory layout of a plan with CS CTAs per repetition (D in shared memory when the
// rings keep stages of >= 4 rows of the wider layout); false if nothing fits
template <int RB>
static bool plan_layout(const DenseAls& a, int CS, ClLayout* out, int* dsh_out) {
  const int rowmax = pitch4(a.nI > a.nJ ? a.nI : a.nJ);
  const int slice_fl = rowmax * (a.nI > a.nJ ? a.nJ : a.nI);
  int dsh = -1;
  for (int d = getenv("SAMBATEN_ALS_GLOBAL_D") ? 0 : 1; d >= 0 && dsh < 0; --d) {
    const ClLayout L0 = cl_layout(a.nI, a.nJ, a.nK, RB, CS, 4, d);
    const size_t fixed = L0.stage;   // the rings are the last region of the layout
    if (fixed + sizeof(float) * 4 * RB * kCT > kSmemCap) continue;
    int sfl = (int)((kSmemCap - fixed) / (sizeof(float) * kTS * L0.NT)) & ~3;
    if (sfl > ((slice_fl + 3) & ~3)) sfl = (slice_fl + 3) & ~3;
    if (sfl > 12288) sfl = 12288;
    if (d == 1 && sfl < 4 * rowmax) continue;
    const ClLayout L = cl_layout(a.nI, a.nJ, a.nK, RB, CS, sfl, d);
    if (L.total <= kSmemCap) { dsh = d; *out = L; }
  }
  *dsh_out = dsh;
  return dsh >= 0;
}

// cost model: a team (warp group) streams whole slices; ~8 busy warps saturate an SM's issue
// slots, so a CTA's pass time ~ nu / min(busy teams * warps per team, 8) * warps per team
static double plan_cost(const ClLayout& L, int nK, int CS, double waves) {
  const int nu = (nK + CS - 1) / CS;
  const int wpt = L.T / 32;
  const int busy = nu < L.NT ? nu : L.NT;
  const double rate = (double)(busy * wpt < 8 ? busy * wpt : 8) / wpt;   // slices in parallel
  return waves * (double)nu / rate + 1e-3 * waves + 1e-5 * CS;
}

template <int RB>
static bool plan_rb(const DenseAls& a, ClusterPlan* pl) {
  if (a.nI > 2 * kCT || a.nJ > 2 * kCT) return false;
  double best = 1e300;
  bool found = false;
  const char* force = getenv("SAMBATEN_ALS_GRID");   // "0": clusters only, "1": grid only
  const bool try_cluster = !force || force[0] != '1';
  const bool try_grid = !force || force[0] != '0';
  for (int CS = 16; CS >= 1 && try_cluster; --CS) {
    if (CS > a.nK) continue;
    ClLayout L{};
    int dsh = -1;
    if (!plan_layout<RB>(a, CS, &L, &dsh)) continue;
    if (cluster_setup<RB, false>(CS, L.total) != cudaSuccess) { cudaGetLastError(); continue; }
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attr[1];
    fill_cfg(&cfg, attr, CS, 1, L.total, nullptr);
    int act = 0;
    if (cudaOccupancyMaxActiveClusters(&act, als_cluster_kernel<RB, false>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      act = 0;
    }
    if (act < 1) continue;
    const double t = plan_cost(L, a.nK, CS, (double)((a.r + act - 1) / act));
    if (getenv("SAMBATEN_DEBUG"))
      fprintf(stderr, "[sambaten]   plan candidate cluster CS=%d act=%d NT=%d T=%d smem=%zu dsh=%d sfl=%d t=%.3f\n",
              CS, act, L.NT, L.T, L.total, dsh, L.stage_fl, t);
    if (t < best) {
      best = t;
      found = true;
      *pl = ClusterPlan{};
      pl->CS = CS; pl->smem = L.total; pl->act = act; pl->RB = RB; pl->stage_fl = L.stage_fl; pl->dsh = dsh;
    }
  }
  if (try_grid) {
    // one co-resident grid, CS = (SMs that hold a CTA) / r CTAs per repetition
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int CS = nsm / a.r;
    if (CS > a.nK) CS = a.nK;
    ClLayout L{};
    int dsh = -1;
    for (; CS >= 2; --CS)
      if (plan_layout<RB>(a, CS, &L, &dsh)) break;
    if (CS >= 2 && cluster_setup<RB, true>(CS, L.total) == cudaSuccess) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, als_cluster_kernel<RB, true>, kCT, L.total);
      cudaGetLastError();
      if (per_sm >= 1 && CS * a.r <= per_sm * nsm) {
        // The per-repetition barriers go through L2 (~1-2 us each, five per iteration), which
        // the passes amortise only when a CTA streams enough slices: the grid is taken when it
        // puts >= 1.25x the SMs of the best cluster plan to work and every CTA owns >= 8
        // slices (measured: C4 summaries 300 x 300 x 320, r = 16: cluster 96 SMs 34.9 ms,
        // grid 144 SMs 24.7 ms; C2 100 x 100 x 100, r = 8: cluster 80 SMs 1.33 ms, grid 144
        // SMs 1.36 ms)
        const double t = plan_cost(L, a.nK, CS, 1.0);
        const int nu = (a.nK + CS - 1) / CS;
        const int cl_sms = found ? pl->CS * (a.r < pl->act ? a.r : pl->act) : 0;
        const bool take = (force && force[0] == '1') || (CS * a.r >= 1.25 * cl_sms && nu >= 8);
        if (getenv("SAMBATEN_DEBUG"))
          fprintf(stderr, "[sambaten]   plan candidate grid CS=%d NT=%d T=%d smem=%zu dsh=%d sfl=%d t=%.3f take=%d\n",
                  CS, L.NT, L.T, L.total, dsh, L.stage_fl, t, (int)take);
        if (take) {
          best = t;
          found = true;
          *pl = ClusterPlan{};
          pl->CS = CS; pl->smem = L.total; pl->act = a.r; pl->RB = RB; pl->stage_fl = L.stage_fl; pl->dsh = dsh;
          pl->grid = 1;
        }
      } else {
        cudaGetLastError();
      }
    } else {
      cudaGetLastError();
    }
  }
  return found;
}

bool plan_als_cluster(const DenseAls& a, ClusterPlan* pl) {
  if (a.r < 1 || a.nI < 1 || a.nJ < 1 || a.nK < 1 || !a.Yt) return false;
  switch (rb_of(a.R)) {
    case 4: return plan_rb<4>(a, pl);
    case 8: return plan_rb<8>(a, pl);
    case 10: return plan_rb<10>(a, pl);
    case 12: return plan_rb<12>(a, pl);
    case 16: return plan_rb<16>(a, pl);
    case 24: return plan_rb<24>(a, pl);
    default: return plan_rb<32>(a, pl);
  }
}

// grid communication buffers after the D scratch: exported P | Gp | sc per CTA, pushed rows,
// barrier counters
static GridComm grid_comm_layout(const DenseAls& a, const ClusterPlan& pl, char* base, size_t* bytes) {
  GridComm g{};
  const int nmax = a.nI > a.nJ ? a.nI : a.nJ;
  g.offP = 0;
  g.offG = nmax * pl.RB;
  g.offS = g.offG + 3 * pl.RB * pl.RB;
  g.xstride = (g.offS + 64 + 31) & ~31;
  g.ustride = (nmax * wstride(pl.RB) + 63) & ~63;
  const size_t xb = sizeof(double) * (size_t)a.r * pl.CS * g.xstride;
  const size_t ub = sizeof(float) * (size_t)a.r * 2 * g.ustride;
  const size_t bb = sizeof(unsigned) * 64 * ((a.r + 63) / 64);
  if (bytes) *bytes = xb + ub + bb + 256;
  if (base) {
    g.x = reinterpret_cast<double*>(base);
    g.u = reinterpret_cast<float*>(base + xb);
    g.bar = reinterpret_cast<unsigned*>(base + xb + ub);
  }
  return g;
}

static size_t d_scratch_bytes(const DenseAls& a, const ClusterPlan& pl) {
  return pl.dsh ? 256 : ((sizeof(float) * (size_t)a.r * ((size_t)a.nK + pl.CS) * a.nJ * pl.RB + 255) & ~(size_t)255);
}

size_t als_cluster_dscratch_bytes(const DenseAls& a, const ClusterPlan& pl) {
  size_t gb = 0;
  if (pl.grid) grid_comm_layout(a, pl, nullptr, &gb);
  return d_scratch_bytes(a, pl) + gb;
}

int cluster_pitch(int n) { return pitch4(n); }

#ifdef SBT_ALS_PHASES
void als_phase_dump() {
  unsigned long long h[32];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, g_als_phase, sizeof(h));
  fprintf(stderr, "[sambaten] als phases (cycles, rank 0 of rep 0):");
  for (int k = 0; k < 32; ++k) fprintf(stderr, " %d:%llu", k, h[k]);
  fprintf(stderr, "\n");
  memset(h, 0, sizeof(h));
  cudaMemcpyToSymbol(g_als_phase, h, sizeof(h));
}
#else
void als_phase_dump() {}
#endif

template <int RB>
static cudaError_t cluster_launch(const DenseAls& a, const ClusterPlan& pl, float* Dglob,
                                  cudaStream_t st) {
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr[1];
  const int narrow = getenv("SAMBATEN_ALS_NARROW_A") ? 2 : 0;
  if (pl.grid) {
    GridComm gc = grid_comm_layout(a, pl, reinterpret_cast<char*>(Dglob) + d_scratch_bytes(a, pl), nullptr);
    cudaError_t e = cudaMemsetAsync(gc.bar, 0, sizeof(unsigned) * a.r, st);
    if (e != cudaSuccess) return e;
    fill_cfg(&cfg, attr, pl.CS, a.r, pl.smem, st, true);
    return cudaLaunchKernelEx(&cfg, als_cluster_kernel<RB, true>, a, pl.CS, Dglob, pl.stage_fl, pl.dsh | narrow, gc);
  }
  fill_cfg(&cfg, attr, pl.CS, a.r, pl.smem, st);
  return cudaLaunchKernelEx(&cfg, als_cluster_kernel<RB, false>, a, pl.CS, Dglob, pl.stage_fl, pl.dsh | narrow,
                            GridComm{});
}

cudaError_t run_als_cluster(const DenseAls& a, const ClusterPlan& pl, float* Dglob, cudaStream_t st) {
  switch (pl.RB) {
    case 4: return cluster_launch<4>(a, pl, Dglob, st);
    case 8: return cluster_launch<8>(a, pl, Dglob, st);
    case 10: return cluster_launch<10>(a, pl, Dglob, st);
    case 12: return cluster_launch<12>(a, pl, Dglob, st);
    case 16: return cluster_launch<16>(a, pl, Dglob, st);
    case 24: return cluster_launch<24>(a, pl, Dglob, st);
    default: return cluster_launch<32>(a, pl, Dglob, st);
  }
}

}  // namespace sbt
