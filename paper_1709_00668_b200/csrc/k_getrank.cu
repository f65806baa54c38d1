// k_getrank.cu -- GetRank quality control (Alg. 2): the
// core consistency diagnostic CorConDia ([bro2003new]) of batched CP models of one dense
// summary (readings R29-R31).  Everything in fp64 (a quality rating, not a hot loop):
//   corcondia_pinv_kernel  block per (model, mode): Gram of the loading matrix (lambda absorbed
//                          into mode 0), its inverse (Gauss-Jordan; pseudo-inverse if singular)
//                          and P_m = Gram^-1 U_m^T (F x n_m) -- pinv for full column rank (R29)
//   corcondia_t1_kernel    T1(f, j, k) = sum_i P_0(f, i) X(i, j, k)
//   corcondia_t2_kernel    T2(f, g, k) = sum_j P_1(g, j) T1(f, j, k)
//   corcondia_core_kernel  G(f, g, h) = sum_k P_2(h, k) T2(f, g, k); cc = 100 (1 - sum (G - T)^2 / F)
#include "als_small.cuh"
#include "common.cuh"
#include "internal.h"

namespace sbt {

namespace {

constexpr int kGT = 256;

struct CcArgs {
  const float* X;  int64_t x_stride, pitch;   // dense [nm][K][J][pitch] (x_stride 0: one tensor)
  int I, J, K, F, nm;                  // nm models
  const float* U[3]; int64_t u_stride[3];   // [nm][n][F] fp32 loadings
  const double* lam;                   // [nm][F]
  double* P;                           // [nm][3][F][nmax]
  double* T1;                          // [nm][F][J][K]
  double* T2;                          // [nm][F][F][K]
  double* W;                           // [nm][3][4][F][F] scratch (Gram, inverse, pinv scratch)
  double* cc;                          // [nm]
  int nmax;
};

__global__ void corcondia_pinv_kernel(CcArgs a) {
  const int mdl = blockIdx.x / 3, m = blockIdx.x % 3;
  const int F = a.F, n = m == 0 ? a.I : m == 1 ? a.J : a.K;
  const float* U = a.U[m] + (int64_t)mdl * a.u_stride[m];
  const double* lam = a.lam + (int64_t)mdl * F;
  double* Gm = a.W + ((int64_t)mdl * 3 + m) * 4 * F * F;
  double* Gi = Gm + F * F;
  double* S1 = Gi + F * F;
  double* S2 = S1 + F * F;
  auto u = [&](int p, int f) { return (double)U[(int64_t)p * F + f] * (m == 0 ? lam[f] : 1.0); };
  for (int e = threadIdx.x; e < F * F; e += blockDim.x) {
    const int f = e / F, g = e - f * F;
    double s = 0.0;
    for (int p = 0; p < n; ++p) s += u(p, f) * u(p, g);
    Gm[e] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // Gauss-Jordan with partial pivoting on [Gm | I]; singular -> pseudo-inverse (pinv_R)
    bool ok = true;
    for (int e = 0; e < F * F; ++e) { S1[e] = Gm[e]; Gi[e] = (e / F == e % F) ? 1.0 : 0.0; }
    double scale = 0.0;
    for (int f = 0; f < F; ++f) scale = fmax(scale, fabs(Gm[f * F + f]));
    for (int c = 0; c < F && ok; ++c) {
      int piv = c;
      for (int rr = c + 1; rr < F; ++rr)
        if (fabs(S1[rr * F + c]) > fabs(S1[piv * F + c])) piv = rr;
      if (!(fabs(S1[piv * F + c]) > 1e-13 * scale)) { ok = false; break; }
      if (piv != c)
        for (int k = 0; k < F; ++k) {
          double t = S1[c * F + k]; S1[c * F + k] = S1[piv * F + k]; S1[piv * F + k] = t;
          t = Gi[c * F + k]; Gi[c * F + k] = Gi[piv * F + k]; Gi[piv * F + k] = t;
        }
      const double inv = 1.0 / S1[c * F + c];
      for (int k = 0; k < F; ++k) { S1[c * F + k] *= inv; Gi[c * F + k] *= inv; }
      for (int rr = 0; rr < F; ++rr)
        if (rr != c) {
          const double fct = S1[rr * F + c];
          if (fct != 0.0)
            for (int k = 0; k < F; ++k) { S1[rr * F + k] -= fct * S1[c * F + k]; Gi[rr * F + k] -= fct * Gi[c * F + k]; }
        }
    }
    if (!ok) pinv_R(Gm, Gi, F, S1, S2);
  }
  __syncthreads();
  double* P = a.P + ((int64_t)mdl * 3 + m) * F * a.nmax;
  for (int e = threadIdx.x; e < F * n; e += blockDim.x) {
    const int f = e / n, p = e - f * n;
    double s = 0.0;
    for (int g = 0; g < F; ++g) s += Gi[f * F + g] * u(p, g);
    P[(int64_t)f * a.nmax + p] = s;
  }
}

__global__ void corcondia_t1_kernel(CcArgs a) {
  const int64_t tot = (int64_t)a.nm * a.F * a.J * a.K;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(e % a.F);
    int64_t r = e / a.F;
    const int j = (int)(r % a.J); r /= a.J;
    const int k = (int)(r % a.K);
    const int mdl = (int)(r / a.K);
    const double* P0 = a.P + ((int64_t)mdl * 3 + 0) * a.F * a.nmax + (int64_t)f * a.nmax;
    const float* x = a.X + mdl * a.x_stride + ((int64_t)k * a.J + j) * a.pitch;
    double s = 0.0;
    for (int i = 0; i < a.I; ++i) s += P0[i] * (double)x[i];
    a.T1[(((int64_t)mdl * a.F + f) * a.J + j) * a.K + k] = s;
  }
}

__global__ void corcondia_t2_kernel(CcArgs a) {
  const int64_t tot = (int64_t)a.nm * a.F * a.F * a.K;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e % a.K);
    int64_t r = e / a.K;
    const int g = (int)(r % a.F); r /= a.F;
    const int f = (int)(r % a.F);
    const int mdl = (int)(r / a.F);
    const double* P1 = a.P + ((int64_t)mdl * 3 + 1) * a.F * a.nmax + (int64_t)g * a.nmax;
    const double* t1 = a.T1 + ((int64_t)mdl * a.F + f) * a.J * a.K + k;
    double s = 0.0;
    for (int j = 0; j < a.J; ++j) s += P1[j] * t1[(int64_t)j * a.K];
    a.T2[(((int64_t)mdl * a.F + f) * a.F + g) * a.K + k] = s;
  }
}

__global__ void corcondia_core_kernel(CcArgs a) {
  __shared__ double red[32];
  const int mdl = blockIdx.x, F = a.F;
  const double* P2 = a.P + ((int64_t)mdl * 3 + 2) * F * a.nmax;
  double dev = 0.0;
  for (int e = threadIdx.x; e < F * F * F; e += blockDim.x) {
    const int h = e % F, g = (e / F) % F, f = e / (F * F);
    const double* t2 = a.T2 + (((int64_t)mdl * F + f) * F + g) * a.K;
    double s = 0.0;
    for (int k = 0; k < a.K; ++k) s += P2[(int64_t)h * a.nmax + k] * t2[k];
    const double d = s - ((f == g && g == h) ? 1.0 : 0.0);
    dev += d * d;
  }
  dev = block_sum_d(dev, red);
  if (threadIdx.x == 0) a.cc[mdl] = 100.0 * (1.0 - dev / F);
}

// Sparse CorConDia ("exploits sparsity"): T1 and T2 are formed from the canonical COO
// (sorted by (k, j, i)) without densifying -- T1(f, j, k) = sum over the fibre (j, k) of
// P_0(f, i) x, T2(f, g, k) = sum_j P_1(g, j) T1(f, j, k) -- by one block per (model, slice k)
// that walks the slice's fibres in order (deterministic): nnz * F + fibres * F^2 work instead
// of I J K F.  The core kernel is the dense one.
struct CcCoo {
  const int32_t *ci, *cj, *ck; const float* cv; int64_t nnz;
};

__global__ void corcondia_t2_coo_kernel(CcArgs a, CcCoo x) {
  extern __shared__ double t1[];   // [F]
  const int k = blockIdx.x % a.K, mdl = blockIdx.x / a.K;
  const int F = a.F;
  // the slice's entry range by binary search on the sorted k
  auto lower = [&](int key) {
    int64_t lo = 0, hi = x.nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (x.ck[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  __shared__ int64_t s_b, s_e;
  if (threadIdx.x == 0) { s_b = lower(k); s_e = lower(k + 1); }
  __syncthreads();
  const int64_t b = s_b, e = s_e;
  const double* P0 = a.P + ((int64_t)mdl * 3 + 0) * F * a.nmax;
  const double* P1 = a.P + ((int64_t)mdl * 3 + 1) * F * a.nmax;
  const int f = threadIdx.x / F, g = threadIdx.x - (threadIdx.x / F) * F;   // T2 cell of this thread
  const bool cell = threadIdx.x < F * F;
  double acc = 0.0;
  for (int64_t t = b; t < e;) {
    const int j = x.cj[t];
    int64_t t2 = t;
    while (t2 < e && x.cj[t2] == j) ++t2;   // the fibre (j, k): [t, t2)
    if (threadIdx.x < F) {
      double s = 0.0;
      for (int64_t u = t; u < t2; ++u) s += P0[(int64_t)threadIdx.x * a.nmax + x.ci[u]] * (double)x.cv[u];
      t1[threadIdx.x] = s;
    }
    __syncthreads();
    if (cell) acc += P1[(int64_t)g * a.nmax + j] * t1[f];
    __syncthreads();
    t = t2;
  }
  if (cell) a.T2[(((int64_t)mdl * F + f) * F + g) * a.K + k] = acc;
}

}  // namespace

cudaError_t launch_corcondia_coo(const int32_t* ci, const int32_t* cj, const int32_t* ck, const float* cv,
                                 int64_t nnz, int I, int J, int K, int F, int nm, const float* const U[3],
                                 const int64_t u_stride[3], const double* lam, double* ws, double* cc,
                                 cudaStream_t st) {
  CcArgs a{};
  a.X = nullptr; a.x_stride = 0; a.pitch = 0; a.I = I; a.J = J; a.K = K; a.F = F; a.nm = nm;
  for (int m = 0; m < 3; ++m) { a.U[m] = U[m]; a.u_stride[m] = u_stride[m]; }
  a.lam = lam;
  a.nmax = max(I, max(J, K));
  a.P = ws;
  a.T1 = nullptr;   // not formed: the fibres feed T2 directly
  a.T2 = a.P + (size_t)nm * 3 * F * a.nmax;
  a.W = a.T2 + (size_t)nm * F * F * K;
  a.cc = cc;
  CcCoo x{ci, cj, ck, cv, nnz};
  corcondia_pinv_kernel<<<nm * 3, kGT, 0, st>>>(a);
  const int threads = ((F * F + 31) / 32) * 32;
  corcondia_t2_coo_kernel<<<nm * K, threads < 64 ? 64 : threads, sizeof(double) * F, st>>>(a, x);
  corcondia_core_kernel<<<nm, kGT, 0, st>>>(a);
  return cudaGetLastError();
}

size_t corcondia_coo_ws_doubles(int I, int J, int K, int F, int nm) {
  const int nmax = max(I, max(J, K));
  return (size_t)nm * (3 * (size_t)F * nmax + (size_t)F * F * K + 12 * (size_t)F * F + 1);
}

size_t corcondia_ws_doubles(int I, int J, int K, int F, int nm) {
  const int nmax = max(I, max(J, K));
  return (size_t)nm * (3 * (size_t)F * nmax + (size_t)F * J * K + (size_t)F * F * K + 12 * (size_t)F * F + 1);
}

cudaError_t launch_corcondia(const float* X, int64_t x_stride, int64_t pitch, int I, int J, int K, int F,
                             int nm, const float* const U[3], const int64_t u_stride[3], const double* lam,
                             double* ws, double* cc, cudaStream_t st) {
  CcArgs a{};
  a.X = X; a.x_stride = x_stride; a.pitch = pitch; a.I = I; a.J = J; a.K = K; a.F = F; a.nm = nm;
  for (int m = 0; m < 3; ++m) { a.U[m] = U[m]; a.u_stride[m] = u_stride[m]; }
  a.lam = lam;
  a.nmax = max(I, max(J, K));
  a.P = ws;
  a.T1 = a.P + (size_t)nm * 3 * F * a.nmax;
  a.T2 = a.T1 + (size_t)nm * F * J * K;
  a.W = a.T2 + (size_t)nm * F * F * K;
  a.cc = cc;
  corcondia_pinv_kernel<<<nm * 3, kGT, 0, st>>>(a);
  const auto blocks = [](int64_t n) { return (unsigned)(ceil_div(n, kGT) < kNumSMs * 8 ? ceil_div(n, kGT) : kNumSMs * 8); };
  corcondia_t1_kernel<<<blocks((int64_t)nm * F * J * K), kGT, 0, st>>>(a);
  corcondia_t2_kernel<<<blocks((int64_t)nm * F * F * K), kGT, 0, st>>>(a);
  corcondia_core_kernel<<<nm, kGT, 0, st>>>(a);
  return cudaGetLastError();
}

// ---- GetRank inside the update (R33) -----------------------------------------------------
namespace {
struct PadArgs {
  const float* Us[3]; const double* lams; const double* fits; const int* iters_s; const int* flags_s;
  float* Ud[3]; double* lamd; double* fitd; int* itersd; int* flagsd;
  int64_t n[3]; int Rs, Rd;
};

__global__ void rank_pad_kernel(PadArgs p) {
  const int64_t n0 = p.n[0] * p.Rd, n1 = n0 + p.n[1] * p.Rd, n2 = n1 + p.n[2] * p.Rd;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= n2 + p.Rd; e += (int64_t)gridDim.x * blockDim.x) {
    if (e < n2) {
      const int m = e < n0 ? 0 : e < n1 ? 1 : 2;
      const int64_t o = e - (m == 0 ? 0 : m == 1 ? n0 : n1);
      const int64_t row = o / p.Rd;
      const int f = (int)(o - row * p.Rd);
      p.Ud[m][o] = f < p.Rs ? p.Us[m][row * p.Rs + f] : 0.0f;
    } else if (e < n2 + p.Rd) {
      const int f = (int)(e - n2);
      p.lamd[f] = f < p.Rs ? p.lams[f] : 0.0;
    } else {
      p.fitd[0] = p.fits[0]; p.itersd[0] = p.iters_s[0]; p.flagsd[0] = p.flags_s[0];
    }
  }
}
}  // namespace

cudaError_t launch_rank_pad(const DenseAls& src, const DenseAls& dst, int rho, cudaStream_t st) {
  PadArgs p{};
  for (int m = 0; m < 3; ++m) {
    p.Us[m] = src.U[m];
    p.Ud[m] = dst.U[m] + rho * dst.u_stride[m];
  }
  p.n[0] = dst.nI; p.n[1] = dst.nJ; p.n[2] = dst.nK;
  p.Rs = src.R; p.Rd = dst.R;
  p.lams = src.lam; p.fits = src.fit; p.iters_s = src.iters; p.flags_s = src.flags;
  p.lamd = dst.lam + (int64_t)rho * dst.R; p.fitd = dst.fit + rho; p.itersd = dst.iters + rho;
  p.flagsd = dst.flags + rho;
  const int64_t tot = (p.n[0] + p.n[1] + p.n[2]) * p.Rd + p.Rd + 1;
  const int64_t nb = ceil_div(tot, kGT);
  rank_pad_kernel<<<(unsigned)(nb < kNumSMs * 4 ? nb : kNumSMs * 4), kGT, 0, st>>>(p);
  return cudaGetLastError();
}

// ---- warm start (R34) ------------------------------------------------------------------------
namespace {
__global__ void warm_init_kernel(DenseAls a, const float* A, const float* B, const float* C, const float* lam,
                                 const int32_t* Is, const int32_t* Js, const int32_t* Kp, int nKs, int rep0,
                                 int rep_stride) {
  const int rep = blockIdx.y, m = blockIdx.z, R = a.R;
  const int n = m == 0 ? a.nI : m == 1 ? a.nJ : a.nK;
  float* U = a.U[m] + rep * a.u_stride[m];
  // the sample lists hold every repetition; local rep `rep` is global repetition rep0 + rep * rep_stride
  const int32_t* idx = (m == 0 ? Is : m == 1 ? Js : Kp) + (int64_t)(rep0 + rep * rep_stride) * n;
  const float* F = m == 0 ? A : m == 1 ? B : C;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)n * R;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e / R), f = (int)(e - (int64_t)row * R);
    float v;
    if (m < 2) v = F[(int64_t)idx[row] * R + f];
    else v = row < nKs ? C[(int64_t)idx[row] * R + f] * lam[f] : 0.0f;
    U[e] = v;
  }
}
}  // namespace

cudaError_t launch_warm_init(const DenseAls& a, const float* A, const float* B, const float* C, const float* lam,
                             const int32_t* Is, const int32_t* Js, const int32_t* Kp, int nKs, cudaStream_t st,
                             int rep0, int rep_stride) {
  const int nmax = max(a.nI, max(a.nJ, a.nK));
  const unsigned gx = (unsigned)ceil_div((int64_t)nmax * a.R, kGT);
  warm_init_kernel<<<dim3(gx < 64 ? gx : 64, a.r, 3), kGT, 0, st>>>(a, A, B, C, lam, Is, Js, Kp, nKs, rep0,
                                                                    rep_stride);
  return cudaGetLastError();
}

}  // namespace sbt
