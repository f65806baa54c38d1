// k_coo.cu -- the sparse (COO) variant of the hot path.
//
//   a0  validation of a canonical batch (sorted by (k,j,i), unique, nonzero, in range; R28)
//       and append into the store's capacity with k shifted by K_old;
//   a3  summaries X(I_s, J_s, K') of all r repetitions in one pass over the nnz:
//       per-mode membership bitmaps (bit rho = sampled in repetition rho) -> per-entry rep
//       mask -> order-preserving two-pass compaction (ballot ranks), relabelled to local
//       coordinates (p, q, u).  The input order (k,j,i) maps to (u,q,p) monotonically, so every
//       summary comes out canonical without a sort;
//   a4  per-mode row structure for the ALS: a stable LSD radix sort (8-bit digits, warp
//       match_any ranks -> deterministic) of each summary by its mode-0 / mode-1 index, row
//       pointers by histogram + scan; MTTKRP with one warp per output row, lanes over the
//       row's entries and a fixed butterfly -> deterministic, no float atomics;
//   a7  fit of the model over the whole COO store.
// All integer work (counts, ranks, offsets) is exact; the gathered values are bit copies.
#include <stdlib.h>

#include "common.cuh"
#include "coo_piece.cuh"
#include "internal.h"

namespace sbt {

namespace {

constexpr int kCT = 256;

// ---------------------------------------------------------------------------------------
// a0: validation and append
// ---------------------------------------------------------------------------------------
__global__ void coo_validate_kernel(const int32_t* __restrict__ ii, const int32_t* __restrict__ jj,
                                    const int32_t* __restrict__ kk, const float* __restrict__ vv,
                                    int64_t n, int64_t I, int64_t J, int64_t K, unsigned* flags) {
  unsigned f = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = ii[e], j = jj[e], k = kk[e];
    if (i < 0 || i >= I || j < 0 || j >= J || k < 0 || k >= K) f |= 1u;   // index range
    const float v = vv[e];
    if (v == 0.0f || !(fabsf(v) <= 3.4e38f)) f |= 2u;                     // zero / non-finite
    if (e + 1 < n) {
      const int32_t i2 = ii[e + 1], j2 = jj[e + 1], k2 = kk[e + 1];
      const bool less = k < k2 || (k == k2 && (j < j2 || (j == j2 && i < i2)));
      if (!less) f |= 4u;                                                 // order / duplicate
    }
  }
  if (f) atomicOr(flags, f);
}

// (may run in place: bi == si etc.)
__global__ void coo_append_kernel(const int32_t* bi, const int32_t* bj, const int32_t* bk,
                                  const float* bv, int64_t n, int32_t k_shift, int32_t* si,
                                  int32_t* sj, int32_t* sk, float* sv) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    si[e] = bi[e];
    sj[e] = bj[e];
    sk[e] = bk[e] + k_shift;
    sv[e] = bv[e];
  }
}

// ---------------------------------------------------------------------------------------
// exclusive scan of int64 (small arrays: up to a few million) -- 3 kernels
// ---------------------------------------------------------------------------------------
constexpr int kScanTile = 2048;

__global__ void scan_tile_kernel(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ out,
                                 int64_t* __restrict__ tile_sums) {
  __shared__ int64_t sh[kCT];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  constexpr int PER = kScanTile / kCT;
  int64_t v[PER];
  int64_t s = 0;
#pragma unroll
  for (int t = 0; t < PER; ++t) {
    const int64_t e = base + threadIdx.x * PER + t;
    v[t] = e < n ? in[e] : 0;
    s += v[t];
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < kCT; o <<= 1) {   // Hillis-Steele inclusive scan of the thread sums
    const int64_t x = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += x;
    __syncthreads();
  }
  int64_t run = threadIdx.x > 0 ? sh[threadIdx.x - 1] : 0;
#pragma unroll
  for (int t = 0; t < PER; ++t) {
    const int64_t e = base + threadIdx.x * PER + t;
    if (e < n) out[e] = run;
    run += v[t];
  }
  if (threadIdx.x == kCT - 1) tile_sums[blockIdx.x] = sh[kCT - 1];
}

__global__ void scan_sums_kernel(int64_t* sums, int64_t n) {   // single block, sequential chunks
  __shared__ int64_t sh[kCT];
  int64_t carry = 0;
  for (int64_t b = 0; b < n; b += kCT) {
    const int64_t e = b + threadIdx.x;
    const int64_t v = e < n ? sums[e] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < kCT; o <<= 1) {
      const int64_t x = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += x;
      __syncthreads();
    }
    if (e < n) sums[e] = carry + sh[threadIdx.x] - v;   // exclusive
    carry += sh[kCT - 1];
    __syncthreads();
  }
}

__global__ void scan_add_kernel(int64_t* out, int64_t n, const int64_t* tile_offsets) {
  const int64_t e = (int64_t)blockIdx.x * kScanTile + threadIdx.x;
  const int64_t off = tile_offsets[blockIdx.x];
  for (int t = 0; t < kScanTile / kCT; ++t) {
    const int64_t x = e + (int64_t)t * kCT;
    if (x < n && x < ((int64_t)blockIdx.x + 1) * kScanTile) out[x] += off;
  }
}

}  // namespace

size_t scan_ws_elems(int64_t n) { return (size_t)ceil_div(n > 0 ? n : 1, kScanTile) + 1; }

// out[e] = sum_{e' < e} in[e'] (in and out may not alias); ws: scan_ws_elems(n) int64
cudaError_t exclusive_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* ws, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t tiles = ceil_div(n, kScanTile);
  scan_tile_kernel<<<(unsigned)tiles, kCT, 0, st>>>(in, n, out, ws);
  scan_sums_kernel<<<1, kCT, 0, st>>>(ws, tiles);
  scan_add_kernel<<<(unsigned)tiles, kCT, 0, st>>>(out, n, ws);
  return cudaGetLastError();
}

namespace {

// ---------------------------------------------------------------------------------------
// a3: gather.  Membership bitmaps from the sampling's local-index maps, then the two passes.
// ---------------------------------------------------------------------------------------
__global__ void build_mask_kernel(const int32_t* __restrict__ loc, int64_t n, int r,
                                  uint32_t* __restrict__ mask, int64_t n_all_after, int64_t total) {
  // mask[x] = OR_rho (loc[rho][x] >= 0) << rho for x < n; entries n <= x < total (the new
  // slices of mode 3) belong to every repetition
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    uint32_t m = 0;
    if (x < n) {
      for (int rho = 0; rho < r; ++rho) m |= (loc[(int64_t)rho * n + x] >= 0 ? 1u : 0u) << rho;
    } else {
      m = r == 32 ? 0xffffffffu : ((1u << r) - 1u);
    }
    mask[x] = m;
  }
  (void)n_all_after;
}

constexpr int kGTile = kCT * 8;   // entries per gather block
constexpr int64_t kGatherSmemMax = 212 * 1024;

// Membership of an entry: mI[i] & mJ[j] & mK[k] (bit rho: in repetition rho's summary).  SM: the
// I and J masks (r <= 8: one byte per index) staged in shared memory once per persistent block
// (C5: 200 KB; the uint32 masks in L2 cost one random sector read per entry and mode), mK read
// from global memory (the entries are sorted by k: a slice's word stays in L1).
template <bool SM>
struct GatherMasks {
  const uint32_t *mI, *mJ, *mK;
  const uint8_t* sh;
  int64_t I;
  __device__ __forceinline__ uint32_t operator()(int i, int j, int k) const {
    if (SM) return (uint32_t)(sh[i] & sh[I + j]) & mK[k];
    return mI[i] & mJ[j] & mK[k];
  }
};

template <bool SM>
__device__ __forceinline__ void stage_masks(const uint32_t* mI, const uint32_t* mJ, int64_t I, int64_t J,
                                            uint8_t* sh) {
  if (!SM) return;
  for (int64_t x = threadIdx.x; x < I + J; x += blockDim.x) sh[x] = (uint8_t)(x < I ? mI[x] : mJ[x - I]);
  __syncthreads();
}

// SM: 1024-thread blocks of four independent 256-thread groups (one tile each, named barrier
// per group), so the persistent block keeps 32 warps in flight; else one group per block.
template <bool SM>
__device__ __forceinline__ void group_sync(int g) {
  if (SM) asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(kCT) : "memory");
  else __syncthreads();
}

// pass 1: counts[rho][tile] of entries with bit rho set (persistent blocks over the tiles)
template <bool SM>
__global__ void __launch_bounds__(SM ? 4 * kCT : kCT) coo_gather_count_kernel(const int32_t* __restrict__ ii, const int32_t* __restrict__ jj,
                                        const int32_t* __restrict__ kk, int64_t n,
                                        const uint32_t* __restrict__ mI, const uint32_t* __restrict__ mJ,
                                        const uint32_t* __restrict__ mK, int64_t I, int64_t J, int r,
                                        int64_t nblocks, int64_t* __restrict__ counts) {
  constexpr int G = SM ? 4 : 1;
  constexpr int RM = SM ? 8 : 32;   // repetitions held in registers (SM: r <= 8)
  extern __shared__ uint8_t msh[];
  __shared__ int cnt_all[G][32];
  stage_masks<SM>(mI, mJ, I, J, msh);
  const GatherMasks<SM> mask{mI, mJ, mK, msh, I};
  const int g = threadIdx.x / kCT, tid = threadIdx.x - g * kCT, lane = tid & 31;
  int* cnt = cnt_all[g];
  for (int64_t tile = (int64_t)blockIdx.x * G + g; tile < nblocks; tile += (int64_t)gridDim.x * G) {
    if (tid < 32) cnt[tid] = 0;
    group_sync<SM>(g);
    const int64_t base = tile * kGTile;
    constexpr int PER = kGTile / kCT;
    int ei[PER], ej[PER], ek[PER];
#pragma unroll
    for (int t = 0; t < PER; ++t) {   // all of the thread's loads in flight at once
      const int64_t e = base + (int64_t)t * kCT + tid;
      const bool in = e < n;
      ei[t] = in ? __ldcs(ii + e) : -1;
      ej[t] = in ? __ldcs(jj + e) : 0;
      ek[t] = in ? __ldcs(kk + e) : 0;
    }
    int local[RM];
#pragma unroll
    for (int rho = 0; rho < RM; ++rho) local[rho] = 0;
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const uint32_t m = ei[t] >= 0 ? mask(ei[t], ej[t], ek[t]) : 0u;
#pragma unroll
      for (int rho = 0; rho < RM; ++rho) local[rho] += (int)((m >> rho) & 1u);
    }
#pragma unroll
    for (int rho = 0; rho < RM; ++rho) {
      if (rho >= r) break;
      const int w = (int)__reduce_add_sync(0xffffffffu, (unsigned)local[rho]);
      if (lane == 0 && w) atomicAdd(&cnt[rho], w);
    }
    group_sync<SM>(g);
    if (tid < r) counts[(int64_t)tid * nblocks + tile] = cnt[tid];
    group_sync<SM>(g);
  }
}

// pass 2: write the entries of every repetition in input order at offsets[rho][tile]
template <bool SM>
__global__ void __launch_bounds__(SM ? 4 * kCT : kCT) coo_gather_write_kernel(const int32_t* __restrict__ ii, const int32_t* __restrict__ jj,
                                        const int32_t* __restrict__ kk, const float* __restrict__ vv,
                                        int64_t n, const uint32_t* __restrict__ mI,
                                        const uint32_t* __restrict__ mJ, const uint32_t* __restrict__ mK,
                                        const int32_t* __restrict__ locI, const int32_t* __restrict__ locJ,
                                        const int32_t* __restrict__ locK, int64_t nIall, int64_t nJall,
                                        int64_t Ko, int nKs, int r, int64_t nblocks,
                                        const int64_t* __restrict__ offsets, int32_t* __restrict__ op,
                                        int32_t* __restrict__ oq, int32_t* __restrict__ ou,
                                        float* __restrict__ ov) {
  constexpr int G = SM ? 4 : 1;
  constexpr int RM = SM ? 8 : 32;
  constexpr int NW = kCT / 32;
  constexpr int PER = kGTile / kCT;
  extern __shared__ uint8_t msh[];
  __shared__ int wcnt_all[G][NW][32];
  __shared__ int64_t woff_all[G][NW][32];
  stage_masks<SM>(mI, mJ, nIall, nJall, msh);
  const GatherMasks<SM> mask{mI, mJ, mK, msh, nIall};
  const int g = threadIdx.x / kCT, tid = threadIdx.x - g * kCT;
  const int lane = tid & 31, warp = tid >> 5;
  int (*wcnt)[32] = wcnt_all[g];
  int64_t (*woff)[32] = woff_all[g];
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t tile = (int64_t)blockIdx.x * G + g; tile < nblocks; tile += (int64_t)gridDim.x * G) {
    // each warp owns a contiguous sub-tile of kGTile / NW entries, processed in rounds of 32
    const int64_t base = tile * kGTile + (int64_t)warp * (kGTile / NW);
    uint32_t mm[PER];
    {
      int ei[PER], ej[PER], ek[PER];
#pragma unroll
      for (int t = 0; t < PER; ++t) {   // all loads in flight, then the masks
        const int64_t e = base + (int64_t)t * 32 + lane;
        const bool in = e < n;
        ei[t] = in ? ii[e] : -1;
        ej[t] = in ? jj[e] : 0;
        ek[t] = in ? kk[e] : 0;
      }
#pragma unroll
      for (int t = 0; t < PER; ++t) mm[t] = ei[t] >= 0 ? mask(ei[t], ej[t], ek[t]) : 0u;
    }
    int c[RM];
#pragma unroll
    for (int rho = 0; rho < RM; ++rho) c[rho] = 0;
#pragma unroll
    for (int t = 0; t < PER; ++t)
#pragma unroll
      for (int rho = 0; rho < RM; ++rho) c[rho] += (int)((mm[t] >> rho) & 1u);
#pragma unroll
    for (int rho = 0; rho < RM; ++rho) {
      if (rho >= r) break;
      const int w = (int)__reduce_add_sync(0xffffffffu, (unsigned)c[rho]);
      if (lane == 0) wcnt[warp][rho] = w;
    }
    group_sync<SM>(g);
    if (tid < r) {   // warp offsets within the tile, in warp order
      int64_t run = offsets[(int64_t)tid * nblocks + tile];
      for (int w = 0; w < NW; ++w) { woff[w][tid] = run; run += wcnt[w][tid]; }
    }
    group_sync<SM>(g);
    int64_t pos[RM];
#pragma unroll
    for (int rho = 0; rho < RM; ++rho) pos[rho] = rho < r ? woff[warp][rho] : 0;
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int64_t e = base + (int64_t)t * 32 + lane;
      const uint32_t m = mm[t];
      if (__ballot_sync(0xffffffffu, m != 0) == 0) continue;   // no member among these 32
      int32_t i = 0, j = 0, k = 0;
      float v = 0.f;
      if (m) { i = ii[e]; j = jj[e]; k = kk[e]; v = vv[e]; }
#pragma unroll
      for (int rho = 0; rho < RM; ++rho) {
        if (rho >= r) break;
        const bool in = (m >> rho) & 1u;
        const unsigned b = __ballot_sync(0xffffffffu, in);
        if (in) {
          const int64_t d = pos[rho] + __popc(b & lt);
          op[d] = locI[(int64_t)rho * nIall + i];
          oq[d] = locJ[(int64_t)rho * nJall + j];
          ou[d] = k < Ko ? locK[(int64_t)rho * Ko + k] : nKs + (k - (int32_t)Ko);
          ov[d] = v;
        }
        pos[rho] += __popc(b);
      }
    }
    group_sync<SM>(g);   // woff / wcnt reused by the next tile
  }
}

// ---------------------------------------------------------------------------------------
// stable LSD radix sort of (key, val) pairs, 8-bit digits (used per summary by mode index)
// ---------------------------------------------------------------------------------------
constexpr int kRTile = 4096;          // elements per block
constexpr int kRW = kCT / 32;         // warps per block
constexpr int kRSub = kRTile / kRW;   // contiguous elements per warp

__global__ void radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                  int64_t nblocks, int64_t* __restrict__ hist /* [256][nblocks] */) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRTile;
  for (int t = threadIdx.x; t < kRTile; t += kCT) {
    const int64_t e = base + t;
    if (e < n) atomicAdd(&h[(keys[e] >> shift) & 255u], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

__global__ void radix_scatter_kernel(const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin,
                                     int64_t n, int shift, int64_t nblocks,
                                     const int64_t* __restrict__ offs /* [256][nblocks] excl */,
                                     uint32_t* __restrict__ kout, int32_t* __restrict__ vout) {
  __shared__ int cnt[kRW][256];
  __shared__ int64_t woff[kRW][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kRW * 256; d += kCT) cnt[d / 256][d % 256] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRTile + (int64_t)warp * kRSub;
  const unsigned lt = (1u << lane) - 1u;
  // per-warp digit counts
  for (int t = 0; t < kRSub; t += 32) {
    const int64_t e = base + t + lane;
    const bool ok = e < n;
    const unsigned d = ok ? (kin[e] >> shift) & 255u : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (ok && (peers & lt) == 0) cnt[warp][d] += __popc(peers);   // the lowest lane of each group
    __syncwarp();
  }
  __syncthreads();
  {   // warp offsets per digit: global block offset + earlier warps
    const int d = threadIdx.x;   // kCT == 256 digits
    int64_t run = offs[(int64_t)d * nblocks + blockIdx.x];
    for (int w = 0; w < kRW; ++w) { woff[w][d] = run; run += cnt[w][d]; }
  }
  __syncthreads();
  for (int t = 0; t < kRSub; t += 32) {
    const int64_t e = base + t + lane;
    const bool ok = e < n;
    const uint32_t key = ok ? kin[e] : 0u;
    const unsigned d = ok ? (key >> shift) & 255u : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    int64_t dst = 0;
    if (ok) dst = woff[warp][d] + __popc(peers & lt);
    __syncwarp();
    if (ok && (peers & lt) == 0) woff[warp][d] += __popc(peers);
    __syncwarp();
    if (ok) {
      kout[dst] = key;
      vout[dst] = vin[e];
    }
  }
}

// The same stable pass with the tile ordered by digit in shared memory first: the tile's
// elements of one digit are written as one contiguous run (consecutive threads, consecutive
// destinations) instead of one scattered 4-byte store per element.  Local position of an
// element = (tile elements of smaller digits) + (earlier warps' elements of its digit) + (its
// rank among the warp's lanes of that digit), so the output equals radix_scatter_kernel's.
constexpr int kRPer = kRSub / 32;     // keys per lane held in registers

__global__ void __launch_bounds__(kCT) radix_scatter_local_kernel(
    const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin, int64_t n, int shift,
    int64_t nblocks, const int64_t* __restrict__ offs /* [256][nblocks] excl */,
    uint32_t* __restrict__ kout, int32_t* __restrict__ vout) {
  __shared__ int cnt[kRW][256];       // per-warp digit counts, then per-warp offsets in the digit
  __shared__ uint32_t sk[kRTile];
  __shared__ int32_t sv[kRTile];
  __shared__ int bstart[256];         // tile-local start of each digit
  __shared__ int64_t goff[256];       // global start of this tile's run of each digit
  __shared__ int wsum[kRW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kRW * 256; d += kCT) cnt[d / 256][d % 256] = 0;
  __syncthreads();
  const int64_t tile0 = (int64_t)blockIdx.x * kRTile;
  const int64_t base = tile0 + (int64_t)warp * kRSub;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t kr[kRPer];
#pragma unroll
  for (int u = 0; u < kRPer; ++u) {
    const int64_t e = base + u * 32 + lane;
    kr[u] = e < n ? __ldcs(kin + e) : 0u;
  }
#pragma unroll
  for (int u = 0; u < kRPer; ++u) {
    const bool ok = base + u * 32 + lane < n;
    const unsigned d = ok ? (kr[u] >> shift) & 255u : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (ok && (peers & lt) == 0) cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    const int d = threadIdx.x;   // kCT == 256 digits
    int tot = 0;
    for (int w = 0; w < kRW; ++w) { const int c = cnt[w][d]; cnt[w][d] = tot; tot += c; }
    goff[d] = offs[(int64_t)d * nblocks + blockIdx.x];
    int inc = tot;               // block-wide exclusive scan of the digit totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int add = 0;
    for (int w = 0; w < warp; ++w) add += wsum[w];
    bstart[d] = add + inc - tot;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kRPer; ++u) {
    const int64_t e = base + u * 32 + lane;
    const bool ok = e < n;
    const unsigned d = ok ? (kr[u] >> shift) & 255u : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    int lpos = 0;
    if (ok) lpos = bstart[d] + cnt[warp][d] + __popc(peers & lt);
    __syncwarp();
    if (ok && (peers & lt) == 0) cnt[warp][d] += __popc(peers);
    __syncwarp();
    if (ok) { sk[lpos] = kr[u]; sv[lpos] = __ldcs(vin + e); }
  }
  __syncthreads();
  const int m = n - tile0 < kRTile ? (int)(n - tile0) : kRTile;
  for (int i = threadIdx.x; i < m; i += kCT) {
    const uint32_t key = sk[i];
    const int d = (key >> shift) & 255u;
    const int64_t dst = goff[d] + (i - bstart[d]);
    kout[dst] = key;
    vout[dst] = sv[i];
  }
}

__global__ void iota_kernel(int32_t* v, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    v[e] = (int32_t)e;
}

// composite key rep << kb | idx for the entries of every repetition (offsets off[0..r])
__global__ void make_keys_kernel(const int32_t* __restrict__ idx, const int64_t* __restrict__ off, int r,
                                 int kb, int64_t n, uint32_t* __restrict__ keys) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int rho = 0;
    while (rho + 1 < r && off[rho + 1] <= e) ++rho;
    keys[e] = ((uint32_t)rho << kb) | (uint32_t)idx[e];
  }
}

// ptr[rho][x] = first position (in the sorted order) of the entries of rep rho with index x;
// from the sorted composite keys: counts then scan.
// The keys are sorted, so ptr[x] for the rows x in (row(e-1), row(e)] is e: every row pointer
// written once, no counting (the Zipf-hot rows made per-entry count atomics contend).
__global__ void key_ptr_kernel(const uint32_t* __restrict__ keys, int64_t n, int kb, int64_t rows, int64_t m,
                               int64_t* __restrict__ ptr /* [m = r*rows + 1] */) {
  const uint32_t lo = (1u << kb) - 1u;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = e < n ? (int64_t)(keys[e] >> kb) * rows + (keys[e] & lo) : m - 1;
    const int64_t xp = e > 0 ? (int64_t)(keys[e - 1] >> kb) * rows + (keys[e - 1] & lo) : -1;
    for (int64_t y = xp + 1; y <= x; ++y) ptr[y] = e;   // e == n: the trailing rows up to m - 1
  }
}

// ---------------------------------------------------------------------------------------
// a4: MTTKRP over the COO summaries:  M(row, f) = sum_{e in row} v_e U_a(a_e, f) U_b(b_e, f).
// The entries of each mode are laid out contiguously by row (sorted copies of the other two
// indices and the values), rows are cut into pieces of <= kPiece entries (Zipf-hot rows
// spread over many warps), one warp per piece: lane l takes entries l, l+32, ... (fp32
// products, fp64 per-lane sums) and a fixed butterfly; single-piece rows write M directly,
// multi-piece rows write partials summed in piece order by a fix-up kernel -> deterministic,
// no float atomics.
// ---------------------------------------------------------------------------------------

// every repetition converged: a whole launch of the iteration has nothing to do (one warp vote;
// r <= 32)
__device__ __forceinline__ bool all_reps_done(const int* done, int r) {
  const int lane = threadIdx.x & 31;
  return __all_sync(0xffffffffu, lane >= r || done[lane] != 0);
}

__global__ void piece_count_kernel(const int64_t* __restrict__ ptr, int64_t nrow, int64_t* __restrict__ cnt) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x <= nrow;
       x += (int64_t)gridDim.x * blockDim.x) {
    if (x == nrow) { cnt[x] = 0; continue; }
    const int64_t len = ptr[x + 1] - ptr[x];
    cnt[x] = len <= kPiece ? 1 : (len + kPiece - 1) / kPiece;
  }
}

__global__ void piece_fill_kernel(const int64_t* __restrict__ ptr, const int64_t* __restrict__ pstart,
                                  int64_t nrow, int64_t* __restrict__ pb, int32_t* __restrict__ prow) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nrow;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = pstart[x], n = pstart[x + 1] - s;
    for (int64_t k = 0; k < n; ++k) {
      pb[s + k] = ptr[x] + k * kPiece;
      prow[s + k] = (int32_t)x;
    }
  }
}

// warp pieces (longer than kShortPiece) and short pieces in two lists (any order: every piece
// writes its own output), so the persistent ALS can schedule the long ones first
__global__ void piece_classify_kernel(const int64_t* __restrict__ ptr, const int64_t* __restrict__ pstart,
                                      const int64_t* __restrict__ pb, const int32_t* __restrict__ prow,
                                      int64_t nrow, int32_t* __restrict__ plist, unsigned* nlist) {
  const int64_t P = pstart[nrow];
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const int x = prow[p];
    const int64_t len = min(pb[p] + kPiece, ptr[x + 1]) - pb[p];
    if (len > kShortPiece) plist[atomicAdd(nlist, 1u)] = (int32_t)p;
    else plist[P - 1 - atomicAdd(nlist + 1, 1u)] = (int32_t)p;
  }
}

// sorted copies: sa[t] = ia[perm[t]], sb[t] = ib[perm[t]], sv[t] = v[perm[t]]
__global__ void permute3_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ ia,
                                const int32_t* __restrict__ ib, const float* __restrict__ v, int64_t n,
                                int32_t* __restrict__ sa, int32_t* __restrict__ sb, float* __restrict__ sv) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = perm[t];
    sa[t] = ia[x];
    sb[t] = ib[x];
    sv[t] = v[x];
  }
}

__global__ void permute4_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ ia,
                                const int32_t* __restrict__ ib, const int32_t* __restrict__ ic,
                                const float* __restrict__ v, int64_t n, int32_t* __restrict__ sa,
                                int32_t* __restrict__ sb, int32_t* __restrict__ sc, float* __restrict__ sv) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = perm[t];
    sa[t] = ia[x];
    sb[t] = ib[x];
    sc[t] = ic[x];
    sv[t] = v[x];
  }
}

// One warp per piece (coo_piece.cuh): grid-stride over the pieces of the mode.
template <int RB>
__global__ void coo_mttkrp_piece_kernel(CooAls a, int mode, int64_t npiece_max) {
  const int lane = threadIdx.x & 31;
  if (all_reps_done(a.done, a.r)) return;
  const unsigned dm = __ballot_sync(0xffffffffu, lane < a.r && a.done[lane] != 0);
  const int64_t P = a.plan[mode].pstart[a.plan[mode].nrow];
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (RB <= 16) {   // short pieces two at a time (half-warps)
    for (int64_t q = w0; 2 * q < P; q += nw) coo_pair_mttkrp<RB>(a, mode, q, P, lane, dm);
  } else {
    for (int64_t piece = w0; piece < P; piece += nw) coo_piece_mttkrp<RB>(a, mode, piece, lane, dm);
  }
  (void)npiece_max;
}

// rows with several pieces: sum the piece partials in order
__global__ void coo_piece_fixup_kernel(CooAls a, int mode) {
  if (all_reps_done(a.done, a.r)) return;
  const CooModePlan& pl = a.plan[mode];
  const int rows = mode == 0 ? a.nI : mode == 1 ? a.nJ : a.nK;
  const int R = a.R;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < pl.nrow * R;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = t / R;
    const int f = (int)(t - x * R);
    const int64_t s = pl.pstart[x], n = pl.pstart[x + 1] - s;
    if (n <= 1) continue;
    const int rep = (int)(x / rows), row = (int)(x - (int64_t)rep * rows);
    if (a.done[rep]) continue;
    double sum = 0.0;
    for (int64_t k = 0; k < n; ++k) sum += pl.partial[(s + k) * R + f];
    a.M[mode][(int64_t)rep * a.m_stride[mode] + (int64_t)row * R + f] = sum;
  }
}

// ||Y_rho||^2: block b of rep rho sums a fixed stride of its entries; partials combined in
// block order (ysq holds r results followed by r * kSqBlocks partials).
constexpr int kSqBlocks = 64;
__global__ void coo_sumsq_kernel(const float* __restrict__ v, const int64_t* __restrict__ off, int r,
                                 double* __restrict__ ysq) {
  __shared__ double red[32];
  const int b = blockIdx.x, rep = blockIdx.y;
  double s = 0.0;
  for (int64_t e = off[rep] + (int64_t)b * blockDim.x + threadIdx.x; e < off[rep + 1];
       e += (int64_t)kSqBlocks * blockDim.x) {
    const double x = v[e];
    s += x * x;
  }
  s = block_sum_d(s, red);
  if (threadIdx.x == 0) ysq[r + rep * kSqBlocks + b] = s;
}

__global__ void coo_sumsq_combine_kernel(int r, double* ysq) {
  const int rep = threadIdx.x;
  if (rep >= r) return;
  double s = 0.0;
  for (int b = 0; b < kSqBlocks; ++b) s += ysq[r + rep * kSqBlocks + b];
  ysq[rep] = s;
}

// ---------------------------------------------------------------------------------------
// a7: fit over the COO store: inner = sum_e v_e sum_f lam_f A(i_e,f) B(j_e,f) C(k_e,f), sq
// ---------------------------------------------------------------------------------------
template <int RB>
__global__ void coo_fit_kernel(const int32_t* __restrict__ ii, const int32_t* __restrict__ jj,
                               const int32_t* __restrict__ kk, const float* __restrict__ vv, int64_t n,
                               const float* __restrict__ lam, const float* __restrict__ A,
                               const float* __restrict__ B, const float* __restrict__ C, int R,
                               double* __restrict__ part, const int32_t* __restrict__ kmap) {
  __shared__ double red[32];
  __shared__ float ls[RB];
  if (threadIdx.x < RB) ls[threadIdx.x] = threadIdx.x < R ? lam[threadIdx.x] : 0.f;
  __syncthreads();
  double inner = 0.0, sq = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float v = vv[e];
    const float* a = A + (int64_t)ii[e] * R;
    const float* b = B + (int64_t)jj[e] * R;
    const float* c = C + (int64_t)(kmap ? kmap[kk[e]] : kk[e]) * R;   // kmap: local -> global slice
    float m = 0.f;
#pragma unroll
    for (int f = 0; f < RB; ++f)
      if (f < R) m = fmaf(ls[f] * a[f], b[f] * c[f], m);
    inner += (double)v * (double)m;
    sq += (double)v * (double)v;
  }
  inner = block_sum_d(inner, red);
  sq = block_sum_d(sq, red);
  if (threadIdx.x == 0) { part[2 * blockIdx.x] = inner; part[2 * blockIdx.x + 1] = sq; }
}

// partials and Grams staged in shared memory by the block (coalesced), summed by thread 0 in
// the fixed sequential order
constexpr int kCooCombT = 256;
__global__ void __launch_bounds__(kCooCombT) coo_fit_combine_kernel(const double* part, int nb, const double* G,
                                                                   const float* lam, int R, double* relerr) {
  __shared__ double sp[2 * kNumSMs * 4];
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

inline unsigned grid_for(int64_t n, int per_block = kCT, int cap = kNumSMs * 8) {
  int64_t g = ceil_div(n > 0 ? n : 1, per_block);
  if (g > cap) g = cap;
  return (unsigned)g;
}

}  // namespace

// ---------------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------------
cudaError_t launch_coo_validate(const int32_t* i, const int32_t* j, const int32_t* k, const float* v,
                                int64_t n, int64_t I, int64_t J, int64_t K, unsigned* flags,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  coo_validate_kernel<<<grid_for(n), kCT, 0, st>>>(i, j, k, v, n, I, J, K, flags);
  return cudaGetLastError();
}

cudaError_t launch_coo_append(const int32_t* bi, const int32_t* bj, const int32_t* bk, const float* bv,
                              int64_t n, int32_t k_shift, int32_t* si, int32_t* sj, int32_t* sk,
                              float* sv, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  coo_append_kernel<<<grid_for(n), kCT, 0, st>>>(bi, bj, bk, bv, n, k_shift, si, sj, sk, sv);
  return cudaGetLastError();
}

cudaError_t launch_build_mask(const int32_t* loc, int64_t n, int r, uint32_t* mask, int64_t total,
                              cudaStream_t st) {
  if (total <= 0) return cudaSuccess;
  build_mask_kernel<<<grid_for(total), kCT, 0, st>>>(loc, n, r, mask, 0, total);
  return cudaGetLastError();
}

int64_t coo_gather_blocks(int64_t nnz) { return ceil_div(nnz > 0 ? nnz : 1, kGTile); }

// the shared-memory masks when r <= 8, I + J bytes fit and the store spans many tiles
static bool gather_sm(const CooView& X, int r, int64_t nb) {
  // staging reads 148 x 4 (I + J) B of masks: worth it when the entries' bytes dwarf that
  return r <= 8 && X.I + X.J <= kGatherSmemMax && nb >= 4 * kNumSMs && X.nnz >= 100 * (X.I + X.J) &&
         !getenv("SAMBATEN_COO_GATHER_GLOBAL");
}

cudaError_t launch_coo_gather_count(const CooView& X, const uint32_t* mI, const uint32_t* mJ,
                                    const uint32_t* mK, int r, int64_t* counts, cudaStream_t st) {
  const int64_t nb = coo_gather_blocks(X.nnz);
  if (gather_sm(X, r, nb)) {
    const int smem = (int)((X.I + X.J + 15) & ~15ll);
    cudaFuncSetAttribute(coo_gather_count_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    coo_gather_count_kernel<true><<<kNumSMs, 4 * kCT, smem, st>>>(X.i, X.j, X.k, X.nnz, mI, mJ, mK, X.I, X.J, r, nb,
                                                                counts);
  } else {
    coo_gather_count_kernel<false><<<(unsigned)nb, kCT, 0, st>>>(X.i, X.j, X.k, X.nnz, mI, mJ, mK, X.I, X.J, r, nb,
                                                                   counts);
  }
  return cudaGetLastError();
}

cudaError_t launch_coo_gather_write(const CooView& X, const uint32_t* mI, const uint32_t* mJ,
                                    const uint32_t* mK, const int32_t* locI, const int32_t* locJ,
                                    const int32_t* locK, int64_t Ko, int nKs, int r,
                                    const int64_t* offsets, int32_t* op, int32_t* oq, int32_t* ou,
                                    float* ov, cudaStream_t st) {
  const int64_t nb = coo_gather_blocks(X.nnz);
  if (gather_sm(X, r, nb)) {
    const int smem = (int)((X.I + X.J + 15) & ~15ll);
    cudaFuncSetAttribute(coo_gather_write_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    coo_gather_write_kernel<true><<<kNumSMs, 4 * kCT, smem, st>>>(X.i, X.j, X.k, X.v, X.nnz, mI, mJ, mK, locI, locJ,
                                                                locK, X.I, X.J, Ko, nKs, r, nb, offsets, op, oq,
                                                                ou, ov);
  } else {
    coo_gather_write_kernel<false><<<(unsigned)nb, kCT, 0, st>>>(X.i, X.j, X.k, X.v, X.nnz, mI, mJ, mK, locI, locJ,
                                                                   locK, X.I, X.J, Ko, nKs, r, nb, offsets, op, oq,
                                                                   ou, ov);
  }
  return cudaGetLastError();
}

size_t radix_ws_elems(int64_t n) { return 256 * (size_t)ceil_div(n > 0 ? n : 1, kRTile); }

// Sort the composite keys (rep << kb | idx[e]) stably; perm receives the entry order, keys the
// sorted keys.  ws_keys/ws_vals: n elements each; hist/offs: radix_ws_elems(n) int64 each,
// sws: scan workspace.
cudaError_t launch_coo_permute4(const int32_t* perm, const int32_t* a, const int32_t* b, const int32_t* c,
                                const float* v, int64_t n, int32_t* oa, int32_t* ob, int32_t* oc, float* ov,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  permute4_kernel<<<grid_for(n), kCT, 0, st>>>(perm, a, b, c, v, n, oa, ob, oc, ov);
  return cudaGetLastError();
}

cudaError_t coo_sort_by_index(const int32_t* idx, const int64_t* off, int r, int kb, int64_t n,
                              uint32_t* keys, int32_t* perm, uint32_t* ws_keys, int32_t* ws_vals,
                              int64_t* hist, int64_t* offs, int64_t* sws, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  make_keys_kernel<<<grid_for(n), kCT, 0, st>>>(idx, off, r, kb, n, keys);
  iota_kernel<<<grid_for(n), kCT, 0, st>>>(perm, n);
  int rb = 0;
  while ((1 << rb) < r) ++rb;
  const int bits = kb + rb;   // (rep, index) keys: 2 passes of 8 bits when they fit 16 bits
  const int64_t nb = ceil_div(n, kRTile);
  uint32_t* ka = keys; int32_t* va = perm;
  uint32_t* kb_ = ws_keys; int32_t* vb = ws_vals;
  int passes = 0;
  // SAMBATEN_RADIX_LOCAL: the tile-local scatter (same permutation; measured no faster at C5: the
  // scattered 4-byte stores merge in L2 before they reach DRAM)
  const bool global_scatter = getenv("SAMBATEN_RADIX_LOCAL") == nullptr;
  for (int shift = 0; shift < bits; shift += 8, ++passes) {
    radix_hist_kernel<<<(unsigned)nb, kCT, 0, st>>>(ka, n, shift, nb, hist);
    cudaError_t e = exclusive_scan_i64(hist, 256 * nb, offs, sws, st);
    if (e != cudaSuccess) return e;
    if (global_scatter)
      radix_scatter_kernel<<<(unsigned)nb, kCT, 0, st>>>(ka, va, n, shift, nb, offs, kb_, vb);
    else
      radix_scatter_local_kernel<<<(unsigned)nb, kCT, 0, st>>>(ka, va, n, shift, nb, offs, kb_, vb);
    uint32_t* tk = ka; ka = kb_; kb_ = tk;
    int32_t* tv = va; va = vb; vb = tv;
  }
  if (passes & 1) {   // result is in the workspace: copy back
    cudaMemcpyAsync(keys, ka, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(perm, va, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st);
  }
  return cudaGetLastError();
}

cudaError_t coo_make_keys(const int32_t* idx, const int64_t* off, int r, int kb, int64_t n,
                          uint32_t* keys, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  make_keys_kernel<<<grid_for(n), kCT, 0, st>>>(idx, off, r, kb, n, keys);
  return cudaGetLastError();
}

// Row pointers from the composite keys (sorted by (rep, index)): ptr = exclusive scan of the
// per-(rep, index) counts, r*rows + 1 entries; rep rho's row x spans [ptr[rho*rows + x],
// ptr[rho*rows + x + 1]).  cnt: r*rows + 1 int64 scratch.
cudaError_t coo_row_pointers(const uint32_t* sorted_keys, int64_t n, int kb, int r, int64_t rows,
                             int64_t* cnt, int64_t* ptr, int64_t* sws, cudaStream_t st) {
  const int64_t m = (int64_t)r * rows + 1;
  (void)cnt; (void)sws;
  key_ptr_kernel<<<grid_for(n + 1), kCT, 0, st>>>(sorted_keys, n, kb, rows, m, ptr);
  return cudaGetLastError();
}

__global__ void coo_max_phi_kernel(const float* __restrict__ v, int64_t n, int moi,
                                   unsigned long long* out) {
  double m = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)v[e];
    m = fmax(m, moi == 0 ? fabs(d) : d * d);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

cudaError_t launch_coo_max_phi(const float* v, int64_t n, int moi, unsigned long long* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  coo_max_phi_kernel<<<grid_for(n), kCT, 0, st>>>(v, n, moi, out);
  return cudaGetLastError();
}

size_t coo_plan_elems(int64_t nrow, int64_t n) { return (size_t)(nrow + n / kPiece + 2); }

// Row pieces of one mode (from its row pointers) and, for the sorted modes, the permuted copies
// of the other two indices and the values.  cnt: nrow+1 int64 scratch, sws: scan workspace.
cudaError_t coo_build_plan(CooModePlan& pl, const int32_t* perm, const int32_t* ia, const int32_t* ib,
                           const float* v, int64_t n, int64_t* cnt, int64_t* sws, cudaStream_t st) {
  piece_count_kernel<<<grid_for(pl.nrow + 1), kCT, 0, st>>>(pl.ptr, pl.nrow, cnt);
  cudaError_t e = exclusive_scan_i64(cnt, pl.nrow + 1, pl.pstart, sws, st);
  if (e != cudaSuccess) return e;
  piece_fill_kernel<<<grid_for(pl.nrow), kCT, 0, st>>>(pl.ptr, pl.pstart, pl.nrow, pl.pb, pl.prow);
  if (pl.plist) {
    e = cudaMemsetAsync(pl.nlist, 0, 2 * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    piece_classify_kernel<<<grid_for(pl.nrow + pl.n / kPiece + 1), kCT, 0, st>>>(pl.ptr, pl.pstart, pl.pb, pl.prow,
                                                                                 pl.nrow, pl.plist, pl.nlist);
  }
  if (perm && n > 0)
    permute3_kernel<<<grid_for(n), kCT, 0, st>>>(perm, ia, ib, v, n, const_cast<int32_t*>(pl.sa),
                                                const_cast<int32_t*>(pl.sb), const_cast<float*>(pl.sv));
  return cudaGetLastError();
}

cudaError_t launch_coo_mttkrp(const CooAls& a, int mode, cudaStream_t st) {
  const CooModePlan& pl = a.plan[mode];
  const int64_t pmax = (int64_t)coo_plan_elems(pl.nrow, pl.n);
  int64_t blocks = ceil_div(pmax * 32, kCT);
  if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
  switch (a.RB) {
    case 4: coo_mttkrp_piece_kernel<4><<<(unsigned)blocks, kCT, 0, st>>>(a, mode, pmax); break;
    case 8: coo_mttkrp_piece_kernel<8><<<(unsigned)blocks, kCT, 0, st>>>(a, mode, pmax); break;
    case 12: coo_mttkrp_piece_kernel<12><<<(unsigned)blocks, kCT, 0, st>>>(a, mode, pmax); break;
    case 16: coo_mttkrp_piece_kernel<16><<<(unsigned)blocks, kCT, 0, st>>>(a, mode, pmax); break;
    case 24: coo_mttkrp_piece_kernel<24><<<(unsigned)blocks, kCT, 0, st>>>(a, mode, pmax); break;
    default: coo_mttkrp_piece_kernel<32><<<(unsigned)blocks, kCT, 0, st>>>(a, mode, pmax); break;
  }
  coo_piece_fixup_kernel<<<grid_for(pl.nrow * a.R), kCT, 0, st>>>(a, mode);
  return cudaGetLastError();
}

cudaError_t launch_coo_sumsq(const float* v, const int64_t* off, int r, double* ysq, cudaStream_t st) {
  coo_sumsq_kernel<<<dim3(kSqBlocks, r), kCT, 0, st>>>(v, off, r, ysq);
  coo_sumsq_combine_kernel<<<1, 32, 0, st>>>(r, ysq);
  return cudaGetLastError();
}

size_t coo_fit_ws_doubles(int64_t I, int64_t J, int64_t K) {
  return 2 * (size_t)kNumSMs * 4 + 3 * kMaxR * kMaxR + 8 + gram3_ws_doubles(I, J, K, kMaxR);
}

static cudaError_t coo_fit_parts(const CooView& X, const float* lam, const float* A, const float* B,
                                 const float* C, int R, const int32_t* kmap, double* ws, int nb, cudaStream_t st) {
  switch (R <= 4 ? 4 : R <= 8 ? 8 : R <= 12 ? 12 : R <= 16 ? 16 : R <= 24 ? 24 : 32) {
    case 4: coo_fit_kernel<4><<<nb, kCT, 0, st>>>(X.i, X.j, X.k, X.v, X.nnz, lam, A, B, C, R, ws, kmap); break;
    case 8: coo_fit_kernel<8><<<nb, kCT, 0, st>>>(X.i, X.j, X.k, X.v, X.nnz, lam, A, B, C, R, ws, kmap); break;
    case 12: coo_fit_kernel<12><<<nb, kCT, 0, st>>>(X.i, X.j, X.k, X.v, X.nnz, lam, A, B, C, R, ws, kmap); break;
    case 16: coo_fit_kernel<16><<<nb, kCT, 0, st>>>(X.i, X.j, X.k, X.v, X.nnz, lam, A, B, C, R, ws, kmap); break;
    case 24: coo_fit_kernel<24><<<nb, kCT, 0, st>>>(X.i, X.j, X.k, X.v, X.nnz, lam, A, B, C, R, ws, kmap); break;
    default: coo_fit_kernel<32><<<nb, kCT, 0, st>>>(X.i, X.j, X.k, X.v, X.nnz, lam, A, B, C, R, ws, kmap); break;
  }
  return cudaGetLastError();
}

__global__ void coo_sum_parts_kernel(const double* part, int nb, double* out2) {
  if (threadIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int i = 0; i < nb; ++i) { a += part[2 * i]; b += part[2 * i + 1]; }
  out2[0] = a;
  out2[1] = b;
}

// sharded fit: this rank's (<X, M>, ||X||^2) over its local store (k local, kmap to global C rows)
cudaError_t launch_coo_fit_partial(const CooView& X, const float* lam, const float* A, const float* B,
                                   const float* C, int R, const int32_t* kmap, double* ws, double* out2,
                                   cudaStream_t st) {
  const int nb = kNumSMs * 4;
  if (X.nnz <= 0) return cudaMemsetAsync(out2, 0, 2 * sizeof(double), st);
  cudaError_t e = coo_fit_parts(X, lam, A, B, C, R, kmap, ws, nb, st);
  if (e != cudaSuccess) return e;
  coo_sum_parts_kernel<<<1, 32, 0, st>>>(ws, nb, out2);
  return cudaGetLastError();
}

cudaError_t launch_coo_fit(const CooView& X, const float* lam, const float* A, const float* B,
                           const float* C, int R, double* ws, double* relerr, cudaStream_t st) {
  const int nb = kNumSMs * 4;
  double* G = ws + 2 * nb;
  cudaError_t e = coo_fit_parts(X, lam, A, B, C, R, nullptr, ws, nb, st);
  if (e != cudaSuccess) return e;
  e = launch_gram3(A, B, C, X.I, X.J, X.K, R, G, G + 3 * kMaxR * kMaxR, st);
  if (e != cudaSuccess) return e;
  coo_fit_combine_kernel<<<1, kCooCombT, 0, st>>>(ws, nb, G, lam, R, relerr);
  return cudaGetLastError();
}

}  // namespace sbt
