// lrbms_affine.cuh -- NEXT-1: the paper's affine online variant of the reduced system (a2 replaced).
//
//   eq:parameterizedMob: lambda_alpha(s) ~ sum_q theta_q(s) lambda_{alpha,q}, with M
//       saturation-independent mobility profiles;
//   eq:leastSquaresFit: Theta(s) = argmin || lambda_t(s) - sum_q theta_q lambda_{t,q} ||_l2
//       over the fine degrees of freedom (k = 0: cells), solved through the normal equations
//       G theta = h, G_qr = <lambda_q, lambda_r> (formed once with the profiles), h_q = <lambda_t(s), lambda_q>;
//   eq:reducedSystem: (c + sum_q theta_q b_q) p_H = e + sum_q theta_q d_q, where b_q, d_q are
//       the projections of the operator / right-hand side of lambda_{t,q} (offline, by k_project), and
//       c = e = 0 under reading R2 (the k = 0 operator and its Dirichlet data are linear in lambda).
//
// Per step: k_theta_partials (one pass over lambda and the M profiles, fixed-order per-CTA partials),
// k_theta_solve (a warp per profile: fixed-order sums; then the substitutions with the Cholesky factor of G
// formed once by k_theta_factor, with dropped pivots for dependent profiles -- the paper's first and last
// profiles are both constant fields), and
// k_affine_combine (blocks = sum_q theta_q b_q, r = sum_q theta_q d_q: a streaming pass over the M
// precomputed operators, HBM-bound).  Deterministic: no atomics.
#pragma once
#include "lrbms_kernels.cuh"

namespace lrbms {

constexpr int AFF_MAXM = 16;

// part[q][blockIdx] = sum over this CTA's cells of x_i * Y[q][i], q < M (grid-stride over cells)
__global__ void __launch_bounds__(256) k_theta_partials(const double* __restrict__ x, const double* __restrict__ Y,
                                                        int M, size_t n, double* __restrict__ part) {
  __shared__ double red[8][AFF_MAXM];
  double acc[AFF_MAXM];
#pragma unroll
  for (int q = 0; q < AFF_MAXM; ++q) acc[q] = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  if ((n & 1) == 0) {   // two cells per thread and 16-byte loads (every profile starts 16-byte aligned)
    const size_t h = n >> 1;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const double2* Y2 = reinterpret_cast<const double2*>(Y);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < h; i += stride) {
      const double2 xi = __ldg(x2 + i);
#pragma unroll
      for (int q = 0; q < AFF_MAXM; ++q)
        if (q < M) {
          const double2 v = __ldcs(Y2 + (size_t)q * h + i);
          acc[q] = fma(xi.x, v.x, acc[q]);
          acc[q] = fma(xi.y, v.y, acc[q]);
        }
    }
  } else {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      const double xi = x[i];
#pragma unroll
      for (int q = 0; q < AFF_MAXM; ++q)
        if (q < M) acc[q] = fma(xi, Y[(size_t)q * n + i], acc[q]);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < AFF_MAXM; ++q) {
    if (q >= M) break;
    const double v = warp_sum(acc[q]);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < M) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w][threadIdx.x];
    part[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
}

// out[q] = sum_b part[q][b] in a fixed order (one warp; lane-strided, then a fixed shuffle tree)
__device__ __forceinline__ void sum_partials(const double* part, int G, int M, double* out) {
  const int lane = threadIdx.x & 31;
  for (int q = 0; q < M; ++q) {
    double v = 0.0;
    for (int b = lane; b < G; b += 32) v += part[(size_t)q * G + b];
    v = warp_sum(v);
    if (lane == 0) out[q] = v;
  }
}

// one warp: row r of the Gram matrix from the partials
__global__ void k_gram_row(const double* __restrict__ part, int G, int M, double* __restrict__ gram, int r) {
  sum_partials(part, G, M, gram + (size_t)r * M);
}

// Once per set_profiles (one thread): the Cholesky factor of the Gram matrix in index order.  A pivot
// below 1e-12 of its original diagonal entry marks a profile that depends on the previous ones: its
// column is dropped (theta_q = 0), which leaves the fitted mobility sum_q theta_q lambda_q -- the
// least-squares projection -- unchanged.  fac = [L (M x M, row-major)][keep (M, 1.0 / 0.0)].
__global__ void k_theta_factor(const double* __restrict__ gram, int M, double* __restrict__ fac) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double* L = fac;
  double* keep = fac + (size_t)M * M;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) L[i * M + j] = gram[(size_t)i * M + j];
  for (int k = 0; k < M; ++k) {
    double d = L[k * M + k];
    for (int j = 0; j < k; ++j)
      if (keep[j] != 0.0) d -= L[k * M + j] * L[k * M + j];
    const bool kp = d > 1e-12 * gram[(size_t)k * M + k] && d > 0.0;
    keep[k] = kp ? 1.0 : 0.0;
    const double lkk = kp ? sqrt(d) : 0.0;
    for (int i = k + 1; i < M; ++i) {
      double v = L[i * M + k];
      for (int j = 0; j < k; ++j)
        if (keep[j] != 0.0) v -= L[i * M + j] * L[k * M + j];
      L[i * M + k] = kp ? v / lkk : 0.0;
    }
    L[k * M + k] = lkk;
  }
}

// Per step, M warps: warp q sums h_q = <lambda_t(s), lambda_q> from the per-CTA partials in a fixed order
// (lane-strided, then a fixed shuffle tree); then one thread does the two substitutions with the stored
// factor from shared memory (the factorisation itself is done once, k_theta_factor).
__global__ void k_theta_solve(const double* __restrict__ part, int G, int M, const double* __restrict__ fac,
                              double* __restrict__ theta) {
  __shared__ double h[AFF_MAXM], Ls[AFF_MAXM * AFF_MAXM], ks[AFF_MAXM];
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  if (q < M) {
    double v = 0.0;
    for (int b = lane; b < G; b += 32) v += part[(size_t)q * G + b];
    v = warp_sum(v);
    if (lane == 0) h[q] = v;
  }
  for (int i = threadIdx.x; i < M * M; i += blockDim.x) Ls[i] = fac[i];
  for (int i = threadIdx.x; i < M; i += blockDim.x) ks[i] = fac[(size_t)M * M + i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double y[AFF_MAXM], t[AFF_MAXM];
#pragma unroll
  for (int i = 0; i < AFF_MAXM; ++i) {   // L y = h
    if (i >= M) break;
    double v = h[i];
#pragma unroll
    for (int j = 0; j < AFF_MAXM; ++j)
      if (j < i) v -= Ls[i * M + j] * y[j];
    y[i] = ks[i] != 0.0 ? v / Ls[i * M + i] : 0.0;
  }
#pragma unroll
  for (int ii = 0; ii < AFF_MAXM; ++ii) {   // L^T t = y
    const int i = AFF_MAXM - 1 - ii;
    if (i >= M) continue;
    double v = y[i];
#pragma unroll
    for (int j = 0; j < AFF_MAXM; ++j)
      if (j > i && j < M) v -= Ls[j * M + i] * t[j];
    t[i] = ks[i] != 0.0 ? v / Ls[i * M + i] : 0.0;
  }
#pragma unroll
  for (int qq = 0; qq < AFF_MAXM; ++qq)
    if (qq < M) theta[qq] = t[qq];
}

// out[i] = sum_q theta_q X[q * qstride + i] for i < len (the reduced operator or right-hand side), 16-byte
// streaming loads -- one pass over the M precomputed operators.  qstride (elements between profiles)
// is even (profile_stride), so every profile starts 16-byte aligned whatever the parity of len.
__global__ void __launch_bounds__(256) k_affine_combine(const double* __restrict__ X, const double* __restrict__ theta,
                                                        int M, size_t len, size_t qstride, double* __restrict__ out) {
  double th[AFF_MAXM];
#pragma unroll
  for (int q = 0; q < AFF_MAXM; ++q) th[q] = q < M ? theta[q] : 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t h = len >> 1, h2 = qstride >> 1;
  const double2* X2 = reinterpret_cast<const double2*>(X);
#ifndef AFF_UNROLL
#define AFF_UNROLL 2
#endif
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; AFF_UNROLL == 2 && i + stride < h; i += 2 * stride) {   // two grid-strides at once: 2 M loads in flight
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int q = 0; q < AFF_MAXM; ++q)
      if (q < M) {
        const double2 v = __ldcs(X2 + (size_t)q * h2 + i);
        const double2 w = __ldcs(X2 + (size_t)q * h2 + i + stride);
        a0 = fma(th[q], v.x, a0);
        a1 = fma(th[q], v.y, a1);
        b0 = fma(th[q], w.x, b0);
        b1 = fma(th[q], w.y, b1);
      }
    __stcs(reinterpret_cast<double2*>(out) + i, make_double2(a0, a1));
    __stcs(reinterpret_cast<double2*>(out) + i + stride, make_double2(b0, b1));
  }
  for (; i < h; i += stride) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int q = 0; q < AFF_MAXM; ++q)
      if (q < M) {
        const double2 v = __ldcs(X2 + (size_t)q * h2 + i);
        a0 = fma(th[q], v.x, a0);
        a1 = fma(th[q], v.y, a1);
      }
    reinterpret_cast<double2*>(out)[i] = make_double2(a0, a1);
  }
  if ((len & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double a = 0.0;
    for (int q = 0; q < M; ++q) a = fma(th[q], X[(size_t)q * qstride + len - 1], a);
    out[len - 1] = a;
  }
}

}  // namespace lrbms
