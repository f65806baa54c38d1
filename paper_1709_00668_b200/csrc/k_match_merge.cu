// k_match_merge.cu -- a5: anchor congruence and optimal matching (Lemma 1;
// R13-R16, R26) and a6: merge (R17-R20).
#include "common.cuh"
#include "internal.h"

namespace sbt {

constexpr int kMatchThreads = 256;

// Hungarian method (potentials; O(R^3)) maximising sum_f S[f][pi f]; single thread.
__device__ void hungarian_max(const double* S, int R, int* pi) {
  double u[kMaxR + 1], v[kMaxR + 1], minv[kMaxR + 1];
  int p[kMaxR + 1], way[kMaxR + 1];
  bool used[kMaxR + 1];
  for (int j = 0; j <= R; ++j) { u[j] = 0; v[j] = 0; p[j] = 0; way[j] = 0; }
  for (int i = 1; i <= R; ++i) {
    p[0] = i;
    int j0 = 0;
    for (int j = 0; j <= R; ++j) { minv[j] = 1e300; used[j] = false; }
    do {
      used[j0] = true;
      const int i0 = p[j0];
      double delta = 1e300;
      int j1 = 0;
      for (int j = 1; j <= R; ++j) {
        if (!used[j]) {
          const double cur = -S[(i0 - 1) * R + (j - 1)] - u[i0] - v[j];
          if (cur < minv[j]) { minv[j] = cur; way[j] = j0; }
          if (minv[j] < delta) { delta = minv[j]; j1 = j; }
        }
      }
      for (int j = 0; j <= R; ++j) {
        if (used[j]) { u[p[j]] += delta; v[j] -= delta; }
        else minv[j] -= delta;
      }
      j0 = j1;
    } while (p[j0] != 0);
    do {
      const int j1 = way[j0];
      p[j0] = p[j1];
      j0 = j1;
    } while (j0);
  }
  for (int j = 1; j <= R; ++j) pi[p[j] - 1] = j - 1;
}

// The same Hungarian method with the column loops spread over the lanes of one warp
// (lane j - 1 owns column j): the arithmetic per element and the choice of j1 (first column
// of minimal minv, strict <) are those of hungarian_max, so pi is identical.  Shared state
// sh: u, v, minv [kMaxR + 1] doubles; p, way [kMaxR + 1] ints.
__device__ void hungarian_max_warp(const double* S, int R, int* pi, double* u, double* v, int* p,
                                   int* way) {
  const int lane = threadIdx.x & 31;
  const int j = lane + 1;                   // this lane's column (valid if j <= R)
  const bool col = j <= R;
  for (int t = lane; t <= R; t += 32) { u[t] = 0.0; v[t] = 0.0; p[t] = 0; way[t] = 0; }   // R + 1 entries (33 at R = 32)
  __syncwarp();
  for (int i = 1; i <= R; ++i) {
    if (lane == 0) p[0] = i;
    int j0 = 0;
    double minv = 1e300;
    bool used = false;      // lane's column used; column 0 is tracked by used0
    bool used0 = false;
    __syncwarp();
    do {
      if (j0 == 0) used0 = true;
      else if (j == j0) used = true;
      const int i0 = p[j0];
      const double ui0 = u[i0];
      // candidate of this lane
      double cand = 1e300;
      int cj = 0x7fffffff;
      if (col && !used) {
        const double cur = -S[(i0 - 1) * R + (j - 1)] - ui0 - v[j];
        if (cur < minv) { minv = cur; way[j] = j0; }
        cand = minv; cj = j;
      }
      // delta = min over unused columns, first column on ties
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double oc = __shfl_xor_sync(0xffffffffu, cand, o);
        const int oj = __shfl_xor_sync(0xffffffffu, cj, o);
        if (oc < cand || (oc == cand && oj < cj)) { cand = oc; cj = oj; }
      }
      const double delta = cand;
      const int j1 = cj == 0x7fffffff ? 0 : cj;
      __syncwarp();   // every lane has read u[i0], v[j] before the updates
      if (col) {
        if (used) { u[p[j]] += delta; v[j] -= delta; }
        else minv -= delta;
      }
      if (lane == 0 && used0) { u[p[0]] += delta; v[0] -= delta; }
      __syncwarp();
      j0 = j1;
    } while (p[j0] != 0);
    if (lane == 0) {
      do {
        const int j1 = way[j0];
        p[j0] = p[j1];
        j0 = j1;
      } while (j0);
    }
    __syncwarp();
  }
  if (col) pi[p[j] - 1] = j - 1;
  __syncwarp();
}

__device__ __forceinline__ void unrank_perm(long long k, int R, int* perm) {
  int avail[8];
  long long fact[9];
  fact[0] = 1;
  for (int i = 1; i <= R; ++i) fact[i] = fact[i - 1] * i;
  for (int i = 0; i < R; ++i) avail[i] = i;
  int na = R;
  for (int i = 0; i < R; ++i) {
    const long long f = fact[R - 1 - i];
    const int d = (int)(k / f);
    k -= d * f;
    perm[i] = avail[d];
    for (int t = d; t < na - 1; ++t) avail[t] = avail[t + 1];
    --na;
  }
}

// Partial anchor sums of one chunk of kMatchRows sampled rows of one mode and repetition:
// part[rep][mode][chunk][0 .. R*R)      = sum_p old(p,f) cand(p,g)  (anchor rows only, R14)
//                       [R*R .. R*R+R)   = sum_p old(p,f)^2
//                       [R*R+R .. +2R)   = sum_p cand(p,g)^2
// Rows are staged in shared memory; thread per entry sums the chunk's rows in order.
constexpr int kMatchRows = 128;

__global__ void __launch_bounds__(kMatchThreads) match_partial_kernel(MatchArgs m, int nchunk) {
  const int chunk = blockIdx.x, mode = blockIdx.y, rep = blockIdx.z;
  const int R = m.R;
  __shared__ float sor[kMatchRows][kMaxR + 1];
  __shared__ float scr[kMatchRows][kMaxR + 1];
  __shared__ unsigned char anc[kMatchRows];
  const float* F = mode == 0 ? m.A : mode == 1 ? m.B : m.C;
  const int64_t iss = m.is_stride ? m.is_stride : m.nI, jss = m.js_stride ? m.js_stride : m.nJ;
  const int32_t* idx = mode == 0 ? m.Is + (int64_t)rep * iss
                     : mode == 1 ? m.Js + (int64_t)rep * jss : m.Ks + (int64_t)rep * m.ks_stride;
  const int n = mode == 0 ? m.nI : mode == 1 ? m.nJ : m.nKs;
  const float* U = m.U[mode] + rep * m.u_stride[mode];
  const int p0 = chunk * kMatchRows;
  const int nr = max(0, min(kMatchRows, n - p0));
  for (int e = threadIdx.x; e < kMatchRows * R; e += blockDim.x) {
    const int pl = e / R, f = e - pl * R;
    float o = 0.f, c = 0.f;
    if (pl < nr) {
      o = F[(int64_t)idx[p0 + pl] * R + f];
      c = U[(int64_t)(p0 + pl) * R + f];
    }
    sor[pl][f] = o;
    scr[pl][f] = c;
  }
  __syncthreads();
  for (int pl = threadIdx.x; pl < kMatchRows; pl += blockDim.x) {
    bool nz = false;
    for (int f = 0; f < R; ++f) nz |= (sor[pl][f] != 0.0f);
    anc[pl] = (pl < nr && nz) ? 1 : 0;
  }
  __syncthreads();
  const int npair = R * R + 2 * R;
  double* out = m.part + (((int64_t)rep * 3 + mode) * nchunk + chunk) * npair;
  for (int pr = threadIdx.x; pr < npair; pr += blockDim.x) {
    double s = 0.0;
    if (pr < R * R) {
      const int f = pr / R, g = pr - f * R;
      for (int pl = 0; pl < nr; ++pl)
        if (anc[pl]) s += (double)sor[pl][f] * (double)scr[pl][g];
    } else if (pr < R * R + R) {
      const int f = pr - R * R;
      for (int pl = 0; pl < nr; ++pl)
        if (anc[pl]) { const double o = sor[pl][f]; s += o * o; }
    } else {
      const int g = pr - R * R - R;
      for (int pl = 0; pl < nr; ++pl)
        if (anc[pl]) { const double c = scr[pl][g]; s += c * c; }
    }
    out[pr] = s;
  }
}

__global__ void __launch_bounds__(kMatchThreads) match_kernel(MatchArgs m, int nchunk) {
  const int rep = blockIdx.x;
  const int R = m.R;
  __shared__ double Phi[3][kMaxR * kMaxR];
  __shared__ double al[3][kMaxR], an[3][kMaxR];
  __shared__ double S[kMaxR * kMaxR];
  __shared__ double bval[kMatchThreads];
  __shared__ long long bidx[kMatchThreads];
  __shared__ int pi_s[kMaxR];
  __shared__ double hu[kMaxR + 1], hv[kMaxR + 1];
  __shared__ int hp[kMaxR + 1], hway[kMaxR + 1];
  const int npair = R * R + 2 * R;
  for (int mode = 0; mode < 3; ++mode) {
    const double* part = m.part + ((int64_t)rep * 3 + mode) * nchunk * npair;
    for (int pr = threadIdx.x; pr < npair; pr += blockDim.x) {
      double s = 0.0;
      for (int c = 0; c < nchunk; ++c) s += part[(int64_t)c * npair + pr];   // chunk order
      if (pr < R * R) Phi[mode][pr] = s;
      else if (pr < R * R + R) al[mode][pr - R * R] = sqrt(s);
      else an[mode][pr - R * R - R] = sqrt(s);
    }
  }
  __syncthreads();
  for (int pr = threadIdx.x; pr < R * R; pr += blockDim.x) {
    const int f = pr / R, g = pr - f * R;
    double t = 0.0;
    for (int mode = 0; mode < 3; ++mode) {
      const double d = al[mode][f] * an[mode][g];
      const double ph = d > 0.0 ? Phi[mode][pr] / d : 0.0;
      Phi[mode][pr] = ph;
      t += fabs(ph);
    }
    S[pr] = t / 3.0;
  }
  __syncthreads();
  if (R <= 8) {
    // exhaustive search in lexicographic order; first maximum wins (R15)
    long long nperm = 1;
    for (int i = 2; i <= R; ++i) nperm *= i;
    double best = -1e300;
    long long bk = 0x7fffffffffffffffll;
    int perm[8];
    for (long long k = threadIdx.x; k < nperm; k += blockDim.x) {
      unrank_perm(k, R, perm);
      double v = 0.0;
      for (int f = 0; f < R; ++f) v += S[f * R + perm[f]];
      if (v > best) { best = v; bk = k; }
    }
    bval[threadIdx.x] = best;
    bidx[threadIdx.x] = bk;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = bval[0];
      long long k = bidx[0];
      for (int t = 1; t < (int)blockDim.x; ++t)
        if (bval[t] > b || (bval[t] == b && bidx[t] < k)) { b = bval[t]; k = bidx[t]; }
      unrank_perm(k, R, perm);
      for (int f = 0; f < R; ++f) pi_s[f] = perm[f];
    }
  } else {
    if (threadIdx.x < 32) hungarian_max_warp(S, R, pi_s, hu, hv, hp, hway);
  }
  __syncthreads();
  // one thread per old component f (the per-f arithmetic of the former sequential loop);
  // the acceptance minimum and the NaN flag are order-free reductions
  __shared__ double s_sc[kMaxR];
  __shared__ int s_valid[kMaxR];
  if (threadIdx.x < R) {
    const int f = threadIdx.x;
    const int g = pi_s[f];
    m.pi[rep * R + f] = g;
    double lh = m.lamp[rep * R + g];
    bool ok_all = true;
    for (int mode = 0; mode < 3; ++mode) {
      const double sig = Phi[mode][f * R + g] < 0.0 ? -1.0 : 1.0;
      const double a0 = al[mode][f], a1 = an[mode][g];
      const bool ok = a0 > 0.0 && a1 > 0.0;
      m.scale[((int64_t)rep * 3 + mode) * R + f] = ok ? sig * a0 / a1 : 0.0;
      if (ok) lh = lh * sig * a1 / a0; else ok_all = false;
    }
    m.lam_hat[rep * R + f] = ok_all ? lh : 0.0;
    s_sc[f] = S[f * R + g];
    s_valid[f] = !(m.rnew && g >= m.rnew[rep]);   // not matched to a zero padding column (R33)
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double smin = 1e300;
    bool nan = false;
    for (int f = 0; f < R; ++f) {
      if (!s_valid[f]) continue;
      const double sc = s_sc[f];
      if (sc != sc) nan = true;
      smin = fmin(smin, sc);
    }
    m.score_min[rep] = smin;
    m.accepted[rep] = (!nan && smin >= m.tau) ? 1 : 0;
  }
}

int match_chunks(const MatchArgs& m) {
  const int nmax = max(m.nI, max(m.nJ, m.nKs));
  return (nmax + kMatchRows - 1) / kMatchRows;
}

size_t match_part_doubles(const MatchArgs& m) {
  return (size_t)m.r * 3 * match_chunks(m) * (m.R * m.R + 2 * m.R);
}

cudaError_t launch_match(const MatchArgs& m, cudaStream_t st) {
  const int nchunk = match_chunks(m);
  match_partial_kernel<<<dim3(nchunk, 3, m.r), kMatchThreads, 0, st>>>(m, nchunk);
  match_kernel<<<m.r, kMatchThreads, 0, st>>>(m, nchunk);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// merge
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void merge_rows(const MergeArgs& g, int mode, int64_t idx) {
  const int64_t n = mode == 0 ? g.I : mode == 1 ? g.J : g.Ko;
  const int R = g.R;
  if (idx >= n * R) return;
  const int64_t row = idx / R;
  const int f = (int)(idx - row * R);
  const float* Fo = mode == 0 ? g.A : mode == 1 ? g.B : g.C;
  float* Fn = mode == 0 ? g.An : mode == 1 ? g.Bn : g.Cn;
  const int32_t* loc = g.loc[mode];
  double s = 0.0;
  int cnt = 0;
  for (int rep = 0; rep < g.r; ++rep) {
    if (!g.accepted[rep]) continue;
    if (g.rnew && g.pi[rep * R + f] >= g.rnew[rep]) continue;   // no candidate column (R33)
    const int l = loc[(int64_t)rep * n + row];
    if (l < 0) continue;
    const float* U = g.U[mode] + rep * g.u_stride[mode];
    s += g.scale[((int64_t)rep * 3 + mode) * R + f] * (double)U[(int64_t)l * R + g.pi[rep * R + f]];
    ++cnt;
  }
  if (cnt) {
    const float old = Fo[idx];
    if (g.policy == 1 || old == 0.0f) Fn[idx] = (float)(s / cnt);
  }
}

__device__ __forceinline__ void merge_new(const MergeArgs& g, int64_t idx) {
  // per component f: mean over the accepted reps that carry it (all accepted reps unless
  // GetRank reduced a rep's rank, R33); no such rep -> C_new(:, f) = 0, lambda_f unchanged
  const int R = g.R;
  const int f = idx < g.Kn * R ? (int)(idx % R) : (int)(idx - g.Kn * R);
  if (idx >= g.Kn * R + R) return;
  auto carries = [&](int rep) {
    return g.accepted[rep] && !(g.rnew && g.pi[rep * R + f] >= g.rnew[rep]);
  };
  int nacc = 0;
  for (int rep = 0; rep < g.r; ++rep) nacc += carries(rep) ? 1 : 0;
  if (idx < g.Kn * R) {
    const int64_t k = idx / R;
    double s = 0.0;
    for (int rep = 0; rep < g.r; ++rep) {
      if (!carries(rep)) continue;
      const float* U = g.U[2] + rep * g.u_stride[2];
      s += g.scale[((int64_t)rep * 3 + 2) * R + f] * (double)U[(g.nKs + k) * R + g.pi[rep * R + f]];
    }
    g.Cn[(g.Ko + k) * R + f] = nacc ? (float)(s / nacc) : 0.0f;
  } else {
    double s = 0.0;
    for (int rep = 0; rep < g.r; ++rep)
      if (carries(rep)) s += g.lam_hat[rep * R + f];
    g.lamn[f] = nacc ? (float)(((double)g.lam[f] + s / nacc) / 2.0) : g.lam[f];
  }
}

// one launch: blocks [0, b[0]) merge A's rows, [b[0], b[1]) B's, [b[1], b[2]) C's old rows,
// [b[2], b[3]) the new rows of C and lambda
struct MergeBlocks { unsigned b[4]; };
__global__ void merge_kernel(MergeArgs g, MergeBlocks mb) {
  const unsigned blk = blockIdx.x;
  int part = 0;
  while (part < 3 && blk >= mb.b[part]) ++part;
  const unsigned b0 = part == 0 ? 0u : mb.b[part - 1];
  const int64_t idx = (int64_t)(blk - b0) * blockDim.x + threadIdx.x;
  if (part < 3) merge_rows(g, part, idx);
  else merge_new(g, idx);
}

cudaError_t launch_merge(const MergeArgs& g, cudaStream_t st) {
  MergeBlocks mb{};
  unsigned acc = 0;
  for (int mode = 0; mode < 3; ++mode) {
    const int64_t n = mode == 0 ? g.I : mode == 1 ? g.J : g.Ko;
    acc += (unsigned)ceil_div(n * g.R, 256);
    mb.b[mode] = acc;
  }
  acc += (unsigned)ceil_div(g.Kn * g.R + g.R, 256);
  mb.b[3] = acc;
  merge_kernel<<<acc, 256, 0, st>>>(g, mb);
  return cudaGetLastError();
}

}  // namespace sbt
