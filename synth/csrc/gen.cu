// synth/csrc/gen.cu -- on-device generator of the dense planted workloads (SURVEY §8(d) "C4:
// generated on device by a Philox generator (domain GEN; Box-Muller in fp64, rounded to
// fp32), slab by slab").  INPUT TOOLING ONLY: it holds none of SamBaTen's arithmetic and is
// built into its own library (synth/libsynthgen.so), separate from the product library; the
// numpy twin is synth/planted.py:dense_philox_slab.
//
//   X(i,j,k) = fl32( sum_f A(i,f) B(j,f) C(k,f) + sigma * z(i,j,k) )        (fp64 inside)
//
// z: standard normals by Box-Muller from Philox4x32-10(key = seed, counter = (p_lo, p_hi,
// 0, 3 << 24)) for the entry pair p = e >> 1 of the global linear index e = (k J + j) I + i
// (z(2p) = r cos(2 pi u2), z(2p+1) = r sin(2 pi u2), r = sqrt(-2 ln u1), u = (2 m52 + 1) 2^-53
// with m52 from the words (x0, x1) for u1 and (x2, x3) for u2).  The clean sum is evaluated
// f = 0..R-1 with separate rounded multiplies and adds (no FMA contraction).
#include <cstdint>
#include <cuda_runtime.h>

namespace {

struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox(uint64_t key, uint64_t c01, uint32_t c2, uint32_t c3) {
  uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
  uint32_t x0 = (uint32_t)c01, x1 = (uint32_t)(c01 >> 32), x2 = c2, x3 = c3;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, x0), lo0 = 0xD2511F53u * x0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, x2), lo1 = 0xCD9E8D57u * x2;
    const uint32_t n0 = hi1 ^ x1 ^ k0, n1 = lo1, n2 = hi0 ^ x3 ^ k1, n3 = lo0;
    x0 = n0; x1 = n1; x2 = n2; x3 = n3;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return U4{x0, x1, x2, x3};
}

__device__ __forceinline__ double unit(uint32_t a, uint32_t b) {
  const uint64_t m52 = ((uint64_t)a << 20) | (b >> 12);
  return (double)(2 * m52 + 1) * 0x1p-53;
}

__global__ void gen_dense_kernel(float* __restrict__ out, const double* __restrict__ A,
                                 const double* __restrict__ B, const double* __restrict__ C, int64_t I,
                                 int64_t J, int R, int64_t k0, int64_t nk, double sigma, uint64_t seed) {
  const int64_t IJ = I * J;
  const int64_t e0 = k0 * IJ, e1 = (k0 + nk) * IJ;
  const int64_t p0 = e0 >> 1, p1 = (e1 + 1) >> 1;
  for (int64_t p = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < p1;
       p += (int64_t)gridDim.x * blockDim.x) {
    double z[2] = {0.0, 0.0};
    if (sigma != 0.0) {
      const U4 x = philox(seed, (uint64_t)p, 0u, 3u << 24);
      const double u1 = unit(x.x, x.y), u2 = unit(x.z, x.w);
      const double rr = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincospi(2.0 * u2, &sn, &cs);
      z[0] = rr * cs;
      z[1] = rr * sn;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t e = 2 * p + h;
      if (e < e0 || e >= e1) continue;
      const int64_t k = e / IJ, rem = e - k * IJ, j = rem / I, i = rem - j * I;
      const double* a = A + i * R;
      const double* b = B + j * R;
      const double* c = C + k * R;
      double s = 0.0;
      for (int f = 0; f < R; ++f) s = __dadd_rn(s, __dmul_rn(__dmul_rn(a[f], b[f]), c[f]));
      out[e - e0] = (float)__dadd_rn(s, __dmul_rn(sigma, z[h]));
    }
  }
}

}  // namespace

extern "C" {

/* Slab [k0, k0 + nk) of the planted dense tensor into `out` (device, [nk][J][I] fp32, i
 * fastest).  A (I x R), B (J x R), C (K x R, all rows of the final tensor) are DEVICE fp64
 * row-major.  Returns a cudaError_t value (0 = success). */
int synth_dense_slab(float* out, const double* A, const double* B, const double* C, int64_t I, int64_t J,
                     int R, int64_t k0, int64_t nk, double sigma, uint64_t seed, void* stream) {
  if (nk <= 0) return 0;
  const int64_t pairs = ((k0 + nk) * I * J + 1) / 2 - (k0 * I * J) / 2;
  int64_t blocks = (pairs + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  gen_dense_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(out, A, B, C, I, J, R, k0, nk, sigma,
                                                                      seed);
  return (int)cudaGetLastError();
}

}
