// common.cuh -- device helpers shared by the SamBaTen sm_100a kernels.
// (Product code; shares nothing with oracle/.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sbt {

constexpr int kMaxR = 32;      // rank limit (register/smem sizing)
constexpr int kMaxReps = 32;   // r <= 32 (rejected-rep bitmask)
constexpr int kNumSMs = 148;   // B200

// ---------------------------------------------------------------------------------------
// Philox4x32-10 (R6): round (c0,c1,c2,c3) -> (hi(M1 c2)^c1^k0, lo(M1 c2), hi(M0 c0)^c3^k1,
// lo(M0 c0)); key bumped by (W0, W1) between the 10 rounds.
// ---------------------------------------------------------------------------------------
struct U4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    U4 n;
    n.x = (uint32_t)(p1 >> 32) ^ c.y ^ k0;
    n.y = (uint32_t)p1;
    n.z = (uint32_t)(p0 >> 32) ^ c.w ^ k1;
    n.w = (uint32_t)p0;
    c = n;
  }
  return c;
}

enum : uint32_t { kDomainSample = 1u, kDomainAlsInit = 2u, kDomainGen = 3u };

__device__ __forceinline__ uint32_t ctr_word3(uint32_t domain, uint32_t rep, uint32_t mode) {
  return (domain << 24) | (rep << 8) | mode;
}

// u = (2*m52 + 1) * 2^-53, m52 = (x0 << 20) | (x1 >> 12): exact, in (0, 1).
__device__ __forceinline__ double uniform53(uint32_t x0, uint32_t x1) {
  const uint64_t m52 = ((uint64_t)x0 << 20) | (uint64_t)(x1 >> 12);
  return __dmul_rn(__dadd_rn(__dmul_rn((double)m52, 2.0), 1.0), 0x1p-53);
}

// detlog (R7): only correctly rounded IEEE operations (no FMA), so the result is bitwise
// identical to any other implementation of the same operation sequence.
__device__ __forceinline__ double detlog(double u) {
  int e;
  double m = frexp(u, &e);  // exact: u = m * 2^e, m in [0.5, 1)
  if (m < 0x1.6a09e667f3bcdp-1) { m = __dmul_rn(m, 2.0); e -= 1; }
  const double f = __dadd_rn(m, -1.0);
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  double p = 0x1.8618618618618p-4;
  p = __dadd_rn(0x1.af286bca1af28p-4, __dmul_rn(z, p));
  p = __dadd_rn(0x1.e1e1e1e1e1e1ep-4, __dmul_rn(z, p));
  p = __dadd_rn(0x1.1111111111111p-3, __dmul_rn(z, p));
  p = __dadd_rn(0x1.3b13b13b13b14p-3, __dmul_rn(z, p));
  p = __dadd_rn(0x1.745d1745d1746p-3, __dmul_rn(z, p));
  p = __dadd_rn(0x1.c71c71c71c71cp-3, __dmul_rn(z, p));
  p = __dadd_rn(0x1.2492492492492p-2, __dmul_rn(z, p));
  p = __dadd_rn(0x1.999999999999ap-2, __dmul_rn(z, p));
  p = __dadd_rn(0x1.5555555555555p-1, __dmul_rn(z, p));
  p = __dadd_rn(0x1p+1, __dmul_rn(z, p));
  const double P = __dmul_rn(s, p);
  const double ed = (double)e;
  return __dadd_rn(__dmul_rn(ed, 0x1.62e42p-1), __dadd_rn(__dmul_rn(ed, 0x1.fdf473dep-22), P));
}

// ---------------------------------------------------------------------------------------
// Reductions
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of doubles in a fixed order (deterministic). `sh` holds >= 32 doubles.
__device__ __forceinline__ double block_sum_d(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum_d(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = lane < nw ? sh[lane] : 0.0;
    t = warp_sum_d(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// Exclusive block scan of ints (any blockDim <= 1024); returns the exclusive prefix and
// writes the block total to *total.  `sh` holds >= 33 ints.
__device__ __forceinline__ int block_excl_scan(int v, int* sh, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sh[lane] = s;          // inclusive warp prefix
    if (lane == 31) sh[32] = s;
  }
  __syncthreads();
  const int before = (w > 0 ? sh[w - 1] : 0);
  *total = sh[32];
  const int r = before + x - v;
  __syncthreads();
  return r;
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace sbt
