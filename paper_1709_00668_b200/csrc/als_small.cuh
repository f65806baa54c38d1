// als_small.cuh -- R x R fp64 helpers of the ALS normal-equation solve (R12):
// Cholesky factorisation and the Jacobi pseudo-inverse fallback (cutoff R*eps*lambda_max).
#pragma once
#include "common.cuh"

namespace sbt {

static __device__ __forceinline__ bool cholesky_R(const double* V, double* L, int R) {
  for (int i = 0; i < R * R; ++i) L[i] = 0.0;
  for (int j = 0; j < R; ++j) {
    double s = V[j * R + j];
    for (int k = 0; k < j; ++k) s -= L[j * R + k] * L[j * R + k];
    if (!(s > 0.0)) return false;
    const double d = sqrt(s);
    L[j * R + j] = d;
    for (int i = j + 1; i < R; ++i) {
      double t = V[i * R + j];
      for (int k = 0; k < j; ++k) t -= L[i * R + k] * L[j * R + k];
      L[i * R + j] = t / d;
    }
  }
  return true;
}

// Pseudo-inverse of a symmetric R x R matrix by cyclic Jacobi (R12); P receives V^+.
static __device__ __noinline__ void pinv_R(const double* V, double* P, int R, double* W /* R*R */, double* Q /* R*R */) {
  for (int i = 0; i < R * R; ++i) { W[i] = V[i]; Q[i] = 0.0; }
  for (int i = 0; i < R; ++i) Q[i * R + i] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < R; ++i)
      for (int j = i + 1; j < R; ++j) off += W[i * R + j] * W[i * R + j];
    if (off < 1e-300) break;
    for (int p = 0; p < R; ++p)
      for (int q = p + 1; q < R; ++q) {
        const double apq = W[p * R + q];
        if (apq == 0.0) continue;
        const double app = W[p * R + p], aqq = W[q * R + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < R; ++k) {
          const double wkp = W[k * R + p], wkq = W[k * R + q];
          W[k * R + p] = c * wkp - s * wkq;
          W[k * R + q] = s * wkp + c * wkq;
        }
        for (int k = 0; k < R; ++k) {
          const double wpk = W[p * R + k], wqk = W[q * R + k];
          W[p * R + k] = c * wpk - s * wqk;
          W[q * R + k] = s * wpk + c * wqk;
        }
        for (int k = 0; k < R; ++k) {
          const double qkp = Q[k * R + p], qkq = Q[k * R + q];
          Q[k * R + p] = c * qkp - s * qkq;
          Q[k * R + q] = s * qkp + c * qkq;
        }
      }
  }
  double wmax = 0.0;
  for (int i = 0; i < R; ++i) wmax = fmax(wmax, W[i * R + i]);
  const double cut = R * 2.220446049250313e-16 * wmax;
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) {
      double s = 0.0;
      for (int k = 0; k < R; ++k) {
        const double w = W[k * R + k];
        if (w > cut) s += Q[i * R + k] * Q[j * R + k] / w;
      }
      P[i * R + j] = s;
    }
}

// Gauss-Jordan in registers for R <= RB <= 16: lane c < 2R holds column c of [V | I].
template <int RB>
static __device__ __forceinline__ bool gj_reg(const double* V, double* Vi, int R) {
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
      col[j] = col[j] / piv;
#pragma unroll
      for (int i = 0; i < RB; ++i)
        if (i < R && i != j) col[i] = fma(-fcol[i], col[j], col[i]);
    }
  }
  if (ok && lane >= R && lane < 2 * R)
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if (i < R) Vi[i * R + (lane - R)] = col[i];
  return ok;
}

}  // namespace sbt
