// coo_piece.cuh -- the COO summary MTTKRP of one row piece (Alg. 1 l.5: the r summary
// decompositions' M = Y_(m) (U_b (.) U_a), Khatri-Rao rows formed on the fly).  Shared by the
// per-mode kernel (k_coo.cu) and the persistent COO ALS (k_coo_als.cu).
//
// Factor reads are plain (L1-cached) loads, not ld.global.nc: the persistent kernel rewrites U
// between phases, and only the coherent path is ordered by its grid barrier (release / acquire
// at gpu scope); Zipf-hot factor rows stay in L1.
//
// Rows of a mode (all repetitions: x = rep * rows + row) are cut into pieces of <= kPiece
// entries; one warp takes a piece.  Short pieces: lane f < R sums component f over the entries
// in order (fp32 products, fp64 sum).  Longer pieces: lane l takes entries l, l+32, ... (fp32
// lane runs of <= kPiece / 32 products), then a fixed butterfly in fp64.  Single-piece rows
// write M directly, multi-piece rows write their piece partial (summed in piece order by the
// consumer) -> deterministic, no float atomics.
#pragma once
#include "common.cuh"
#include "internal.h"

namespace sbt {

constexpr int kPiece = 256;
constexpr int kShortPiece = 16;   // pieces up to this many entries: lane per component

// done_mask: bit rep set = repetition converged (its pieces are skipped)
template <int RB>
__device__ __forceinline__ void coo_piece_mttkrp(const CooAls& a, int mode, int64_t piece, int lane,
                                                 unsigned done_mask) {
  const CooModePlan& pl = a.plan[mode];
  const int rows = mode == 0 ? a.nI : mode == 1 ? a.nJ : a.nK;
  const int R = a.R;
  const int oa = mode == 0 ? 1 : 0, ob = mode == 2 ? 1 : 2;
  const int x = pl.prow[piece];
  const int rep = x / rows, row = x - rep * rows;
  if ((done_mask >> rep) & 1u) return;
  const int64_t b = pl.pb[piece];
  const int64_t e = min(b + kPiece, pl.ptr[x + 1]);
  const bool single = pl.pstart[x + 1] - pl.pstart[x] == 1;
  double* out = single ? a.M[mode] + (int64_t)rep * a.m_stride[mode] + (int64_t)row * R
                       : pl.partial + piece * R;
  if (e - b <= kShortPiece) {
    if (lane < R) {
      const float* Ua = a.U[oa] + rep * a.u_stride[oa];
      const float* Ub = a.U[ob] + rep * a.u_stride[ob];
      double s = 0.0;
      for (int64_t t = b; t < e; ++t) {
        const float v = __ldcs(pl.sv + t);
        s += (double)(v * Ua[(int64_t)__ldcs(pl.sa + t) * R + lane] * Ub[(int64_t)__ldcs(pl.sb + t) * R + lane]);
      }
      out[lane] = s;
    }
    return;
  }
  if (a.Up[oa]) {
    // padded factor rows (16 B aligned): vector gathers; fp32 lane runs, then per component
    // (double) and a fixed fp64 butterfly -- one component at a time (few live registers)
    const float4* Ua = reinterpret_cast<const float4*>(a.Up[oa] + rep * a.up_stride[oa]);
    const float4* Ub = reinterpret_cast<const float4*>(a.Up[ob] + rep * a.up_stride[ob]);
    float ac[RB];
#pragma unroll
    for (int f = 0; f < RB; ++f) ac[f] = 0.f;
#pragma unroll 2
    for (int64_t t = b + lane; t < e; t += 32) {
      const float v = __ldcs(pl.sv + t);
      const float4* ra = Ua + (int64_t)__ldcs(pl.sa + t) * (RB / 4);
      const float4* rb = Ub + (int64_t)__ldcs(pl.sb + t) * (RB / 4);
#pragma unroll
      for (int f4 = 0; f4 < RB / 4; ++f4) {
        const float4 xa = ra[f4], yb = rb[f4];
        ac[4 * f4 + 0] = fmaf(v * xa.x, yb.x, ac[4 * f4 + 0]);
        ac[4 * f4 + 1] = fmaf(v * xa.y, yb.y, ac[4 * f4 + 1]);
        ac[4 * f4 + 2] = fmaf(v * xa.z, yb.z, ac[4 * f4 + 2]);
        ac[4 * f4 + 3] = fmaf(v * xa.w, yb.w, ac[4 * f4 + 3]);
      }
    }
    double mine = 0.0;
#pragma unroll
    for (int f = 0; f < RB; ++f) {
      double sf = (double)ac[f];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sf += __shfl_xor_sync(0xffffffffu, sf, o);
      if (f == lane) mine = sf;
    }
    if (lane < R) out[lane] = mine;
    return;
  }
  double acc[RB];
  {
    const float* Ua = a.U[oa] + rep * a.u_stride[oa];
    const float* Ub = a.U[ob] + rep * a.u_stride[ob];
#pragma unroll
    for (int f = 0; f < RB; ++f) acc[f] = 0.0;
#pragma unroll 2
    for (int64_t t = b + lane; t < e; t += 32) {
      const float v = __ldcs(pl.sv + t);
      const float* ra = Ua + (int64_t)__ldcs(pl.sa + t) * R;
      const float* rb = Ub + (int64_t)__ldcs(pl.sb + t) * R;
#pragma unroll
      for (int f = 0; f < RB; ++f)
        if (f < R) acc[f] += (double)(v * ra[f] * rb[f]);
    }
  }
#pragma unroll
  for (int f = 0; f < RB; ++f) {
    double s = acc[f];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    acc[f] = s;
  }
  if (lane < R) {
    double v = 0.0;
#pragma unroll
    for (int f = 0; f < RB; ++f)
      if (f == lane) v = acc[f];
    out[lane] = v;
  }
}

// Short piece by a half-warp (R <= 16): lane f = hl < R sums component f over the entries in
// order -- the arithmetic of the warp short path (fp32 products, fp64 sum), four entries' loads
// in flight.  hl: lane within the half-warp.
__device__ __forceinline__ void coo_short_half(const CooAls& a, int mode, int64_t piece, int hl,
                                               unsigned done_mask) {
  const CooModePlan& pl = a.plan[mode];
  const int rows = mode == 0 ? a.nI : mode == 1 ? a.nJ : a.nK;
  const int R = a.R;
  const int oa = mode == 0 ? 1 : 0, ob = mode == 2 ? 1 : 2;
  const int x = pl.prow[piece];
  const int rep = x / rows, row = x - rep * rows;
  if ((done_mask >> rep) & 1u) return;
  if (hl >= R) return;
  const int64_t b = pl.pb[piece];
  const int64_t e = min(b + kPiece, pl.ptr[x + 1]);
  const bool single = pl.pstart[x + 1] - pl.pstart[x] == 1;
  double* out = single ? a.M[mode] + (int64_t)rep * a.m_stride[mode] + (int64_t)row * R
                       : pl.partial + piece * R;
  // the padded copies (rows of RB floats, 16 B aligned) when kept: fewer sectors per row
  const bool pad = a.Up[oa] != nullptr;
  const int rs = pad ? a.RB : R;
  const float* Ua = (pad ? a.Up[oa] + rep * a.up_stride[oa] : a.U[oa] + rep * a.u_stride[oa]) + hl;
  const float* Ub = (pad ? a.Up[ob] + rep * a.up_stride[ob] : a.U[ob] + rep * a.u_stride[ob]) + hl;
  double s = 0.0;
  int64_t t = b;
  for (; t + 4 <= e; t += 4) {
    float v[4], ua[4], ub[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[q] = __ldcs(pl.sv + t + q);
      ua[q] = Ua[(int64_t)__ldcs(pl.sa + t + q) * rs];
      ub[q] = Ub[(int64_t)__ldcs(pl.sb + t + q) * rs];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) s += (double)(v[q] * ua[q] * ub[q]);
  }
  for (; t < e; ++t) s += (double)(__ldcs(pl.sv + t) * Ua[(int64_t)__ldcs(pl.sa + t) * rs] * Ub[(int64_t)__ldcs(pl.sb + t) * rs]);
  out[hl] = s;
}

// Pieces 2 q and 2 q + 1 by one warp (R <= 16): two short pieces go to the two half-warps at
// once; otherwise each piece in turn (a long one by the whole warp).  Results are the same as
// coo_piece_mttkrp's.
template <int RB>
__device__ __forceinline__ void coo_pair_mttkrp(const CooAls& a, int mode, int64_t q, int64_t P, int lane,
                                                unsigned done_mask) {
  const CooModePlan& pl = a.plan[mode];
  const int64_t p0 = 2 * q, p1 = p0 + 1;
  auto is_short = [&](int64_t p) {
    const int x = pl.prow[p];
    const int64_t b = pl.pb[p];
    return min(b + kPiece, pl.ptr[x + 1]) - b <= kShortPiece;
  };
  const bool s0 = is_short(p0);
  const bool s1 = p1 < P && is_short(p1);
  if (s0 && s1) {
    coo_short_half(a, mode, lane < 16 ? p0 : p1, lane & 15, done_mask);
    return;
  }
  if (s0) { if (lane < 16) coo_short_half(a, mode, p0, lane, done_mask); }
  else coo_piece_mttkrp<RB>(a, mode, p0, lane, done_mask);
  if (p1 < P) {
    if (s1) { if (lane < 16) coo_short_half(a, mode, p1, lane, done_mask); }
    else coo_piece_mttkrp<RB>(a, mode, p1, lane, done_mask);
  }
}

}  // namespace sbt
