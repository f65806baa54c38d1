// k_sample.cu -- a2: importance sampling without replacement (Alg. 1 l.3 P:211; R4-R6).
//
// One block per (rep, mode) segment.  key_i = -detlog(u_i) / (double)w_i (+inf if w_i == 0)
// with u_i from Philox4x32-10 (counter (i, 0, update_id, 1<<24 | rep<<8 | mode)).  Positive
// doubles order like their bit patterns, so the n_s-th smallest key T is found by an 8-pass
// MSB radix select on the 64-bit patterns (shared-memory histogram of 256 digits per pass).
// The sample is then compacted in index order: keys < T, plus the first (n_s - #{key < T})
// indices with key == T -- exactly the n_s smallest (key, index) pairs, already sorted.
#include "common.cuh"
#include "internal.h"

namespace sbt {

constexpr int kSampleThreads = 1024;

__global__ void __launch_bounds__(kSampleThreads) sample_kernel(const SampleSeg* __restrict__ segs,
                                                                uint64_t seed, uint32_t update_id) {
  const SampleSeg sg = segs[blockIdx.x];
  __shared__ unsigned hist[256];
  __shared__ int scan_sh[40];
  __shared__ unsigned long long sh_prefix;
  __shared__ long long sh_k;
  const int64_t n = sg.n, ns = sg.ns;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const uint32_t w3 = ctr_word3(kDomainSample, sg.rep, sg.mode);
  // keys
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t w = sg.w[i];
    unsigned long long key = 0x7FF0000000000000ull;  // +inf
    if (w > 0) {
      const U4 o = philox4x32_10(U4{(uint32_t)i, 0u, update_id, w3}, k0, k1);
      const double E = -detlog(uniform53(o.x, o.y));
      key = (unsigned long long)__double_as_longlong(__ddiv_rn(E, __ll2double_rn(w)));
    }
    sg.keys[i] = key;
  }
  if (threadIdx.x == 0) { sh_prefix = 0; sh_k = ns; }
  __syncthreads();
  if (ns <= 0) return;
  // radix select of the ns-th smallest key
  unsigned long long mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[d] = 0;
    __syncthreads();
    const unsigned long long prefix = sh_prefix;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long key = sg.keys[i];
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // the first digit d with (keys below d) + hist[d] >= k, as a warp: lane l holds digits
      // 8l .. 8l+7; an inclusive scan of the lane sums finds the lane, the lane finds d
      const int lane = threadIdx.x;
      const long long k = sh_k;
      long long loc[8], s = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) { loc[t] = hist[lane * 8 + t]; s += loc[t]; }
      long long incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned ball = __ballot_sync(0xffffffffu, incl >= k);
      if (ball && lane == __ffs(ball) - 1) {
        long long cum = incl - s;
        int d = lane * 8 + 7;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (cum + loc[t] >= k) { d = lane * 8 + t; break; }
          cum += loc[t];
        }
        sh_k = k - cum;
        sh_prefix = prefix | ((unsigned long long)d << shift);
      }
    }
    mask |= 0xFFull << shift;
    __syncthreads();
  }
  const unsigned long long T = sh_prefix;
  const long long need_eq = sh_k;   // number of keys == T to take (smallest indices first)
  // ordered compaction
  long long eq_seen = 0, out_pos = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    unsigned long long key = 0xFFFFFFFFFFFFFFFFull;
    if (i < n) key = sg.keys[i];
    const int is_eq = (i < n && key == T) ? 1 : 0;
    int tot_eq;
    const int eq_rank = block_excl_scan(is_eq, scan_sh, &tot_eq);
    const int take = (i < n) && (key < T || (is_eq && eq_seen + eq_rank < need_eq));
    int tot_take;
    const int pos = block_excl_scan(take, scan_sh, &tot_take);
    if (take) sg.out[out_pos + pos] = (int32_t)i;
    if (sg.loc && i < n) sg.loc[i] = take ? (int32_t)(out_pos + pos) : -1;
    eq_seen += tot_eq;
    out_pos += tot_take;
  }
  for (int64_t t = threadIdx.x; t < sg.ntail; t += blockDim.x)
    sg.kp_tail[t] = (int32_t)(sg.tail0 + t);
}

cudaError_t launch_sample(const SampleSeg* segs_dev, int nseg, uint64_t seed, uint32_t update_id,
                          cudaStream_t st) {
  if (nseg <= 0) return cudaSuccess;
  sample_kernel<<<nseg, kSampleThreads, 0, st>>>(segs_dev, seed, update_id);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// test hooks: Philox and detlog on device
// ---------------------------------------------------------------------------------------
__global__ void philox_kernel(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t key,
                              int64_t n, uint32_t* out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const U4 o = philox4x32_10(U4{c0 + (uint32_t)t, c1, c2, c3}, (uint32_t)key, (uint32_t)(key >> 32));
    out[4 * t] = o.x; out[4 * t + 1] = o.y; out[4 * t + 2] = o.z; out[4 * t + 3] = o.w;
  }
}

__global__ void detlog_kernel(const double* u, int64_t n, double* out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = detlog(u[t]);
}

cudaError_t launch_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t key,
                          int64_t n, uint32_t* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t b = ceil_div(n, 256); if (b > 4096) b = 4096;
  philox_kernel<<<(unsigned)b, 256, 0, st>>>(c0, c1, c2, c3, key, n, out);
  return cudaGetLastError();
}

cudaError_t launch_detlog(const double* u, int64_t n, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t b = ceil_div(n, 256); if (b > 4096) b = 4096;
  detlog_kernel<<<(unsigned)b, 256, 0, st>>>(u, n, out);
  return cudaGetLastError();
}

}  // namespace sbt
